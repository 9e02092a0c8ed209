#!/bin/sh
# Build the reference's compiled kernel core (sellkit._kernels) from its own
# source under /root/reference into oracle/_ref/ -- the "reference" CPU arm
# and an extra parity pin.  Mirrors /root/reference/pkg/setup.py:29-42:
# Cython language_level=3, numpy include, NPY_NO_DEPRECATED_API, -O3.
# Outputs only into oracle/_ref/ (git-ignored, travels to the GPU box).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${REF:-/root/reference/pkg/src/sellkit/_kernels.pyx}
PY=${PY:-python3}
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
    echo "build_ref.sh: $SRC not present; keeping prebuilt oracle/_ref" >&2
    exit 0
fi
mkdir -p "$OUT"
cython -3 "$SRC" -o "$OUT/_kernels.c"
EXT=$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
PYINC=$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
NPINC=$($PY -c 'import numpy; print(numpy.get_include())')
gcc -O3 -shared -fPIC -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$PYINC" -I"$NPINC" "$OUT/_kernels.c" -o "$OUT/_kernels$EXT"
echo "built $OUT/_kernels$EXT"
