#!/usr/bin/env bash
# Builds oracle/_ref/_kernel*.so: the reference's own compiled FSE kernel
# (/root/reference/pkg/src/fsefill/_kernel.pyx, i.e. run_fse + _iterate,
# _kernel.pyx:14-187) compiled straight from its single source file with
# cython + gcc, exactly the flags the reference's setup.py:5-12 implies
# (-O3, no -march, so no FMA contraction).  Test/bench infrastructure only:
# the product never imports it.  Outputs go only into oracle/_ref/ (git-ignored;
# travels to the GPU box with the snapshot).  Needs /root/reference, so it is
# run here, never on the GPU box.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/fsefill/_kernel.pyx
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source $SRC not present; skipping oracle/_ref build" >&2
  exit 0
fi
PY=${PYTHON:-python}
mkdir -p "$OUT"
EXT=$($PY -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
PYINC=$($PY -c "import sysconfig; print(sysconfig.get_paths()['include'])")
NPINC=$($PY -c "import numpy; print(numpy.get_include())")
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp "$SRC" "$TMP/_kernel.pyx"
$PY -m cython -3 -o "$TMP/_kernel.c" "$TMP/_kernel.pyx"
gcc -O3 -fwrapv -fno-strict-aliasing -fPIC -shared -w \
    -I"$PYINC" -I"$NPINC" "$TMP/_kernel.c" -o "$OUT/_kernel$EXT"
echo "built $OUT/_kernel$EXT"
