#!/usr/bin/env bash
# Build the PS_DEBUG=1 variant (bounded spin waits that __trap instead of
# hanging) into a scratch directory and run the sanitizer workload on it.
set -euo pipefail
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
DST="${1:-/tmp/ps_debug}"
rm -rf "$DST" && mkdir -p "$DST"
cp -r "$ROOT/paper_2506_15556_b200" "$ROOT/include" "$DST/"
ln -s "$ROOT/baseline" "$DST/baseline"
rm -rf "$DST/paper_2506_15556_b200/_build" "$DST/paper_2506_15556_b200/libpredgen_b200.so"
PS_DEBUG=1 python -c "import sys; sys.path.insert(0, '$DST'); from paper_2506_15556_b200 import build; print(build.build())"
cd "$DST" && python "$ROOT/tools/sanitize_run.py" all
