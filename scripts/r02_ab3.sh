#!/bin/bash
# Round-2 A/B, part 3: group walk with unconditional gathers (grp*u) and
# without the metadata prefetch (grp6n), against the Hybrid ELL walk.
out=${1:-gpurun_out/r02_ab3.txt}
: > "$out"
for p in 4 8; do
  python scripts/ab_formats.py --case 5:2048 --prec $p --rounds 3 --k 100 --variants auto,grp6u,grp6n,hybrid:g6 >> "$out" 2>&1
  python scripts/ab_formats.py --case 5:1024 --prec $p --rounds 3 --k 100 --variants auto,grp6u,grp6n,hybrid:g6 >> "$out" 2>&1
  python scripts/ab_formats.py --case 7:256 --prec $p --rounds 3 --k 100 --variants auto,grp8u,grp8ru,hybrid:litef >> "$out" 2>&1
  python scripts/ab_formats.py --case 27:128 --prec $p --rounds 3 --k 100 --variants auto,grp7u,grp8ru,hybrid:g7 >> "$out" 2>&1
done
