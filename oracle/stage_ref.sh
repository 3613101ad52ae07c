#!/bin/sh
# Stage the reference implementation (triad, pure Python + numpy) as an
# installed build artefact under oracle/_ref/ -- git-ignored, but it travels to
# the GPU box with gpurun, where bench.py times triad's own CPU loss path
# (group_loss + combine_reports, algorithms.py:351-379) as the reference arm /
# cpu_baseline.  The sources stay where they lie under /root/reference: pip
# builds a wheel from a scratch copy (the tree is read-only) and installs it.
# TEST / MEASUREMENT INFRASTRUCTURE ONLY: nothing in the product imports it.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
[ -f "$SRC/pyproject.toml" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --quiet \
    --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import triad.algorithms, triad.policy  # noqa: F401  (the timed path imports)
print("staged", triad.__file__)
PY
