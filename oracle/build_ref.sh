#!/usr/bin/env bash
# Install the LIVE reference package (velreg, pure Python + numba) into
# oracle/_ref so it travels to the GPU box with the repo snapshot (oracle/_ref
# is git-ignored, not gpurun-ignored).  Test / baseline infrastructure only:
# bench.py --impl reference times it, tests may compare against it; the product
# never imports it.  The source tree is copied to /tmp first because the
# setuptools build writes egg-info next to the sources and /root/reference is
# read-only.  Dependencies (numpy, numba) are already in the image: --no-deps.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference sources not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/velreg_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC"/. "$TMP"/
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import velreg
print("oracle/_ref: velreg", getattr(velreg, "__version__", "0.1.0"), "from", velreg.__file__)
PY
