# Interleaved A/B of K2 variants + Hybrid over the stencil shapes (scripts/ab_formats.py).
# usage: bash scripts/k2_ab.sh <variants> [cases]
V=${1:-lite,lite8,lite_mpf,lite8_mpf,lite8_full,lite8_full_mpf,vec2,vec4,hybrid}
CASES=${2:-"5:1024 5:2048 5:4096 7:256 7:384 27:128"}
for c in $CASES; do for p in 8 4; do
timeout 300 python scripts/ab_formats.py --case $c --prec $p --rounds 3 --k 50 --variants $V 2>&1 | grep -v Warn
done; done
