#!/bin/bash
# Installs the UNMODIFIED reference package (dart 0.1.0, pure Python + NumPy) into baseline/_ref
# so that bench.py can time the reference's own code on the GPU box's host cores (the box has no
# /root/reference; baseline/_ref is git-ignored but travels with the gpurun snapshot).
# Test/bench infrastructure only: nothing in paper_2603_11441_b200/ imports it.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${DART_REFERENCE:-/root/reference}/pkg"
DEST="$ROOT/baseline/_ref"
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "install_ref: $SRC not found; skipping (bench falls back to the oracle port)" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"   # the build writes egg-info into the source tree; /root/reference is read-only
rm -rf "$DEST"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$DEST" "$TMP/pkg" >/dev/null
python -c "import sys; sys.path.insert(0, '$DEST'); import dart.model, dart.pipeline; print('install_ref: dart', dart.model.__file__)"
