#!/bin/bash
# Round-2 kernel A/B (scripts/ab_formats.py): Hybrid group-walk shapes on the
# stencils, L2 eviction hints on the power-law paths.  Output: gpurun_out/r02_ab.txt
set -u
out=${1:-gpurun_out/r02_ab.txt}
: > "$out"
for p in 8 4; do
  for c in 27:128 7:256 5:2048; do
    python scripts/ab_formats.py --case $c --prec $p --rounds 3 --k 100 \
      --variants auto,hybrid:litef,hybrid:g6,hybrid:g7,hybrid:g8,hybrid:g8r >> "$out" 2>&1
  done
  python scripts/ab_formats.py --case 0:8000000 --prec $p --rounds 3 --k 20 \
    --variants lite8,lite8h,lite,liteh,pipe,hybrid:litef,hybrid:litefh >> "$out" 2>&1
  SPMVK_LONG_HINT=0 python scripts/ab_formats.py --case 0:8000000 --prec $p --rounds 3 --k 20 \
    --variants pipe,lite8h >> "$out" 2>&1
  python scripts/ab_formats.py --case 0:8000000 --reorder --prec $p --rounds 3 --k 20 \
    --variants pipe,lite8,lite8h,liteh,hybrid:litef,hybrid:litefh >> "$out" 2>&1
  SPMVK_LONG_HINT=0 python scripts/ab_formats.py --case 0:8000000 --reorder --prec $p --rounds 3 \
    --k 20 --variants pipe,lite8h >> "$out" 2>&1
done
