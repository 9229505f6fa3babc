#!/usr/bin/env bash
# Install the UNMODIFIED reference (poseflow, /root/reference/pkg) into
# baseline/_ref — git-ignored, but it travels to the GPU box with gpurun —
# for the bench's reference arm and the drop-in tests.
#   * the package: pip from a /tmp copy (the build writes egg-info into the
#     source tree; /root/reference is read-only); --no-deps because numpy is
#     already in the image and matplotlib (report plots only) is not;
#   * its test suite, next to it (baseline/_ref/poseflow_tests), so the GPU box
#     can run the reference's own tests with paf.parse swapped for the GPU one
#     (tests/test_gpu_reference_dropin.py).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DST"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" "$TMP/pkg" >/dev/null
rm -rf "$DST/poseflow_tests"
cp -r "$SRC/tests" "$DST/poseflow_tests"
rm -rf "$TMP"
python - "$DST" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import poseflow, poseflow.paf
print("installed", poseflow.__file__)
PY
