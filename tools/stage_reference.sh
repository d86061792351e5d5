#!/usr/bin/env bash
# Install the UNMODIFIED reference package (pkg/ of the reference tree) into the
# git-ignored baseline/_ref, the one offline install the task allows:
#   python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
#       --target baseline/_ref <reference>
# setuptools writes build/ and *.egg-info into the source tree, and the reference
# tree is read-only, so the install runs from a copy under /tmp.  --no-deps: the
# only dependency (numpy) is already in the image.  baseline/_ref is git-ignored
# but not gpurun-ignored, so it travels to the GPU host: the -m gpu tests that run
# the reference's own code (tests/test_gpu_reference.py) and `bench.py --impl
# reference` import it from there.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -f "$SRC/pyproject.toml" ] || { echo "no reference package at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
python - "$ROOT/baseline/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import blk.musr, blk.theory, blk.backend
print("baseline/_ref: blk", blk.musr.__file__)
PY
