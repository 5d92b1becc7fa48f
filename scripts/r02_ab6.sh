#!/bin/bash
# Round-2 A/B, part 6: programmatic dependent launch on the fp64 group walk.
out=${1:-gpurun_out/r02_ab6.txt}
: > "$out"
for pdl in 0 1; do
  echo "SPMVK_PDL=$pdl" >> "$out"
  SPMVK_PDL=$pdl python scripts/ab_formats.py --case 27:128 --prec 8 --rounds 5 --k 200 --variants auto,grp8_r64 >> "$out" 2>&1
  SPMVK_PDL=$pdl python scripts/ab_formats.py --case 7:256 --prec 8 --rounds 3 --k 100 --variants auto >> "$out" 2>&1
  SPMVK_PDL=$pdl python scripts/ab_formats.py --case 5:1024 --prec 8 --rounds 3 --k 200 --variants auto,grp8_r64 >> "$out" 2>&1
done
