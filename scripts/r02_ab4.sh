#!/bin/bash
# Round-2 A/B, part 4: Hybrid ELL pitch padding (SPMVK_ELL_PAD=0/1).
out=${1:-gpurun_out/r02_ab4.txt}
: > "$out"
for pad in 0 1; do
  echo "SPMVK_ELL_PAD=$pad" >> "$out"
  for p in 4 8; do
    for c in 27:128 7:256 5:2048; do
      SPMVK_ELL_PAD=$pad python scripts/ab_formats.py --case $c --prec $p --rounds 3 --k 100 --variants auto,hybrid >> "$out" 2>&1
    done
    SPMVK_ELL_PAD=$pad python scripts/ab_formats.py --case 0:8000000 --prec $p --rounds 3 --k 20 --variants auto,hybrid >> "$out" 2>&1
  done
  SPMVK_ELL_PAD=$pad python scripts/probes/hyb_probe.py >> "$out" 2>&1
done
