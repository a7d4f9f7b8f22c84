#!/usr/bin/env bash
# Install the reference package `specstream` (pure Python, /root/reference/pkg)
# into baseline/_ref, unmodified. The source tree is read-only, so the build
# runs from a copy under /tmp. No network: --no-index, and numpy (its only
# dependency) is already in the image, hence --no-deps.
set -euo pipefail
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "reference package not found at $SRC" >&2
  exit 1
fi
TMP="$(mktemp -d /tmp/specstream_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC/." "$TMP/"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP"
python - "$ROOT/baseline/_ref" <<'EOF'
import sys
sys.path.insert(0, sys.argv[1])
import specstream
print("installed specstream", specstream.__version__, "->", specstream.__file__)
EOF
