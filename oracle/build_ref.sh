#!/usr/bin/env bash
# Build the UNMODIFIED reference `mrsolve` package (Python + one Cython
# kernel file) into oracle/_ref/ so it can serve as the CPU baseline arm
# (`bench.py --impl reference`) and as a cross-check for the oracle port.
#
# TEST INFRASTRUCTURE ONLY: nothing in paper_2103_07329_b200/ imports this.
#
# Recipe (mirrors /root/reference/pkg/setup.py:5-14 without running its build
# system): cythonize src/mrsolve/kernels/_ckernels.pyx from where it lies,
# compile the generated C with gcc -O2 (CPython's default extension flags, no
# -march, so no FMA -- the reference's arithmetic), and place the pure-Python
# modules next to it.  Outputs go only to oracle/_ref/ (git-ignored).
set -euo pipefail
REF=${REF:-/root/reference/pkg}
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
if [ ! -d "$REF/src/mrsolve" ]; then
  echo "build_ref: $REF not present; keeping prebuilt $OUT" >&2
  exit 0
fi
PY=${PYTHON:-python3}
rm -rf "$OUT"; mkdir -p "$OUT/build"
# pure-Python modules of the package (runtime copy; never committed)
cp -r "$REF/src/mrsolve" "$OUT/mrsolve"
find "$OUT/mrsolve" -name '__pycache__' -prune -exec rm -rf {} +
rm -f "$OUT"/mrsolve/kernels/*.so "$OUT"/mrsolve/kernels/_ckernels.c
"$PY" -m cython -3 -o "$OUT/build/_ckernels.c" "$REF/src/mrsolve/kernels/_ckernels.pyx"
INC_PY=$("$PY" -c 'import sysconfig;print(sysconfig.get_paths()["include"])')
INC_NP=$("$PY" -c 'import numpy;print(numpy.get_include())')
SUFFIX=$("$PY" -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')
gcc -O2 -fwrapv -fno-strict-aliasing -DNDEBUG -fPIC -shared \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$INC_PY" -I"$INC_NP" "$OUT/build/_ckernels.c" \
    -o "$OUT/mrsolve/kernels/_ckernels$SUFFIX"
echo "built $OUT/mrsolve (kernels backend: cython)"
