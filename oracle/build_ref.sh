#!/usr/bin/env bash
# Build the UNMODIFIED reference (`stasim`, /root/reference/pkg/src/stasim) into
# oracle/_ref/ so it can travel to the GPU box as the CPU baseline / checker.
#
# TEST INFRASTRUCTURE ONLY: nothing in paper_2603_28381_b200/ imports oracle/.
#
# Recipe (no reference build system is run):
#   1. copy the reference's Python sources into oracle/_ref/stasim/ (git-ignored
#      build output, never committed);
#   2. cython -> C for _kernels.pyx, then gcc with the reference's own flags
#      (-O2 -ffp-contract=off, /root/reference/pkg/setup.py:21-23) into
#      oracle/_ref/stasim/_kernels<EXT_SUFFIX>.
# If /root/reference is absent (the GPU box) this is a no-op: the prebuilt
# oracle/_ref/ shipped with the repo snapshot is used as is.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC=/root/reference/pkg/src/stasim
OUT="$HERE/_ref/stasim"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC not present; using prebuilt $OUT" >&2
  exit 0
fi
PY=${PYTHON:-python}
EXT=$($PY -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
if [ -f "$OUT/_kernels$EXT" ] && [ "$OUT/_kernels$EXT" -nt "$SRC/_kernels.pyx" ]; then
  exit 0
fi
mkdir -p "$OUT/data"
cp "$SRC"/*.py "$OUT/"
cp "$SRC"/data/*.json "$OUT/data/"
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp "$SRC/_kernels.pyx" "$TMP/_kernels.pyx"
$PY -m cython -3 "$TMP/_kernels.pyx" -o "$TMP/_kernels.c" >/dev/null
PYINC=$($PY -c "import sysconfig; print(sysconfig.get_paths()['include'])")
NPINC=$($PY -c "import numpy; print(numpy.get_include())")
gcc -O2 -ffp-contract=off -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$PYINC" -I"$NPINC" "$TMP/_kernels.c" -o "$OUT/_kernels$EXT"
echo "build_ref: built $OUT/_kernels$EXT" >&2
