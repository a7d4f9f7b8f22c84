"""ORACLE — test infrastructure, not product.

CPU restatements used only as the checker by tests/, `__graft_entry__.smoke()`
and the `cpu_baseline` / `--impl reference` legs of bench.py:

* `weights`  — the counter-based weight generator (bit-identical to csrc/init.cu)
* `decoder`  — float64 numpy decoder + `CpuDecoderLM`, a reference
               `LanguageModel` (`/root/reference/pkg/src/specstream/lm.py:157-213`)

The algorithm layer is the reference's own package (`specstream`, installed
into baseline/_ref by tools/install_reference.sh), so the oracle has no copy
of it. Decoder numerics are parity-unpinned by the reference (it has no
decoder); the algorithm layer is pinned by golden event logs the reference
itself produced (tests/golden/make_golden.py).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

_REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
try:
    specstream = importlib.import_module("specstream")
except ImportError:
    if str(_REF) not in sys.path:
        sys.path.append(str(_REF))
    specstream = importlib.import_module("specstream")
