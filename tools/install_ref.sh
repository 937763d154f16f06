#!/usr/bin/env bash
# Install the unmodified reference (hybridann 0.1.0) into the git-ignored baseline/_ref/ so
# that the GPU box can run the reference's own test suite with its kernel module swapped for
# ours (tests/test_ref_swap.py).  baseline/_ref/ is git-ignored (not product source) but not
# gpurun-ignored, so it travels with the snapshot.  Run here, where /root/reference exists.
#   baseline/_ref/site   pip --target install of /root/reference/pkg (no deps: numpy, numba
#                        and scipy are in the image)
#   baseline/_ref/tests  the reference's tests (not part of the wheel)
#   baseline/_ref/test_output.txt  the reference's recorded run (acceptance numbers)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"            # the build writes egg-info into the source tree
rm -rf "$DST"
mkdir -p "$DST"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$DST/site" "$TMP/pkg"
cp -r "$SRC/tests" "$DST/tests"
cp "$SRC/test_output.txt" "$DST/test_output.txt"
echo "installed $(ls "$DST/site")"
