#!/usr/bin/env bash
# Compiles the reference's own compiled blend kernel (splatnav/raster/_kernels_cy.pyx) from
# its source under /root/reference into oracle/_ref/ (git-ignored build output). Used only to
# pin the C oracle's blend loop bit-for-bit against the reference (tests/golden/make_golden.py).
# No reference source is copied into the repo; cython writes its generated C into _ref/.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/splatnav/raster/_kernels_cy.pyx
OUT="$HERE/_ref"
PY="${PYTHON:-python}"
[ -f "$SRC" ] || { echo "reference source not present; skipping"; exit 0; }
mkdir -p "$OUT"
"$PY" -m cython -3 -o "$OUT/_kernels_cy.c" "$SRC"
INC="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
EXT="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
# same optimisation level the reference's setup.py requests (-O3), no -march: no FMA contraction
${CC:-gcc} -O3 -fPIC -shared -I"$INC" "$OUT/_kernels_cy.c" -o "$OUT/_kernels_cy$EXT"
echo "built $OUT/_kernels_cy$EXT"
