#!/bin/sh
# Test infrastructure: install the UNMODIFIED reference package (pure Python,
# /root/reference/pkg) into oracle/_ref so it travels to the GPU box with the
# repo snapshot (oracle/_ref is git-ignored, not gpurun-ignored).  Only the
# tests, bench.py's reference arm / cpu_baseline and smoke() import it -- as the
# CLIENT of the drop-in (ref_adapter.py) and as the CPU reference being timed.
# The reference tree is read-only, so the build runs from a copy under /tmp.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
if [ ! -d "$SRC" ]; then
  echo "build_ref: no reference at $SRC (GPU box?) -- keeping the prebuilt oracle/_ref"
  exit 0
fi
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-deps --no-build-isolation --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import hpgalerkin, hpgalerkin.assembly, hpgalerkin.proximal, hpgalerkin.linalg  # noqa
print("build_ref: hpgalerkin", hpgalerkin.__version__, "->", hpgalerkin.__file__)
PY
