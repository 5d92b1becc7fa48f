#!/bin/bash
# Round-2 A/B, part 2: one more resident CTA per SM for the fp32 group walk;
# the long-row kernel overlapped with the thread-per-row kernel.
out=${1:-gpurun_out/r02_ab2.txt}
: > "$out"
python scripts/ab_formats.py --case 5:2048 --prec 4 --rounds 3 --k 100 --variants auto,grp6o,hybrid:g6 >> "$out" 2>&1
python scripts/ab_formats.py --case 7:256 --prec 4 --rounds 3 --k 100 --variants auto,grp8o,grp7o,hybrid:litef >> "$out" 2>&1
python scripts/ab_formats.py --case 27:128 --prec 4 --rounds 3 --k 100 --variants auto,grp7o,grp8o,hybrid:g7 >> "$out" 2>&1
python scripts/ab_formats.py --case 5:1024 --prec 4 --rounds 3 --k 100 --variants auto,grp6o,hybrid:g6 >> "$out" 2>&1
for ov in 0 1; do
  echo "SPMVK_LONG_OVERLAP=$ov" >> "$out"
  SPMVK_LONG_OVERLAP=$ov python scripts/ab_formats.py --case 0:8000000 --reorder --prec 8 --rounds 3 --k 20 --variants pipe >> "$out" 2>&1
  SPMVK_LONG_OVERLAP=$ov python scripts/ab_formats.py --case 0:8000000 --reorder --prec 4 --rounds 3 --k 20 --variants pipe >> "$out" 2>&1
  SPMVK_LONG_OVERLAP=$ov python scripts/ab_formats.py --case 0:8000000 --prec 8 --rounds 3 --k 20 --variants lite8 >> "$out" 2>&1
  SPMVK_LONG_OVERLAP=$ov python scripts/ab_formats.py --case 0:8000000 --prec 4 --rounds 3 --k 20 --variants pipe >> "$out" 2>&1
done
