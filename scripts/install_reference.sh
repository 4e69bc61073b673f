#!/usr/bin/env bash
# Install the UNMODIFIED reference package `voxgrid` (/root/reference/pkg) into
# baseline/_ref for the CPU baseline and `bench.py --impl reference`.
# Offline: the build runs from a copy under /tmp (the reference tree is
# read-only), no index, no build isolation; --no-deps because its runtime
# dependencies (numpy, scikit-learn) are already in the image. baseline/_ref is
# git-ignored but not gpurun-ignored, so it travels to the GPU box.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "reference not present ($SRC): nothing to install"; exit 0; }
TMP="$(mktemp -d /tmp/voxgrid_ref.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
PYTHONPATH="$ROOT/baseline/_ref" python -c "import voxgrid, sys; print('installed', voxgrid.__file__)"
