"""Locate the reference package `specstream` (the algorithm layer this backend plugs into).

The predict-and-verify loop itself — `run_turn`, `run_baseline`,
`verify_greedy`, `ar_generate`, `SentenceTracker`, `compute_metrics`, the
SimClock and the TTS latency model — is the reference's own code, used
unmodified. It is installed (not copied) into `baseline/_ref/` by
`tools/install_reference.sh`
(`pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>`);
`__graft_entry__.build()` runs that recipe when the directory is missing.
`baseline/_ref/` is git-ignored but travels with the gpurun snapshot, so the
GPU box imports the same installed package.

An already-importable `specstream` (e.g. a maintainer's own install) wins.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_TARGET = ROOT / "baseline" / "_ref"


class ReferenceNotInstalledError(ImportError):
    pass


def load():
    try:
        return importlib.import_module("specstream")
    except ImportError:
        pass
    if (REF_TARGET / "specstream" / "__init__.py").exists():
        if str(REF_TARGET) not in sys.path:
            sys.path.append(str(REF_TARGET))
        return importlib.import_module("specstream")
    raise ReferenceNotInstalledError(
        "the reference package `specstream` is not importable and baseline/_ref is empty; "
        "run tools/install_reference.sh (or __graft_entry__.build()) in a container that has /root/reference")


specstream = load()
