mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hybrid.py -x -q 2>&1 | tail -3
for c in 27:128 7:256 5:2048 0:8000000; do for p in 8 4; do
timeout 300 python scripts/ab_formats.py --case $c --prec $p --rounds 3 --k 50 --variants auto,hybrid:v4,hybrid:lite,hybrid:lite8,hybrid:lite8_full 2>&1 | grep -v Warn
done; done
