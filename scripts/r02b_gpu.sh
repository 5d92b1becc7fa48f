# Round 2 (second session) evidence pass on one B200: GPU suite, bench (both
# arms), ncu of the fused long-row kernel (config 3, both orders, fp64) and of
# the fp32 Hybrid power-law kernel (x L2 residency), sanitizer over the new
# paths.  usage: bash scripts/r02b_gpu.sh <tag> [skip-tests]
TAG=${1:-r02b}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; tail -1 $O/smoke_$TAG.log
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_$TAG.log 2>&1; tail -3 $O/pytest_$TAG.log
fi
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; tail -c 400 $O/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2>&1; tail -c 200 $O/bench_ref_$TAG.json
for ro in "" "--reorder"; do
  t=pl8m_f64${ro:+_desc}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rgcsr_spmv" -s 2 -c 1 \
    -o $O/prof_${TAG}_$t python scripts/prof_k2.py --case 0:8000000:32 --prec 8 --variant auto \
    --format rgcsr $ro > $O/ncu_${TAG}_$t.log 2>&1; tail -1 $O/ncu_${TAG}_$t.log
done
for p in 4 8; do
  timeout 900 ncu --set full --clock-control none -k regex:"hybrid_spmv" -s 2 -c 1 \
    -o $O/prof_${TAG}_hyb_pl8m_p$p python scripts/prof_k2.py --case 0:8000000:32 --prec $p \
    --format hybrid > $O/ncu_${TAG}_hyb_p$p.log 2>&1; tail -1 $O/ncu_${TAG}_hyb_p$p.log
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py > $O/san_${TAG}_$tool.log 2>&1
  tail -2 $O/san_${TAG}_$tool.log
done
ls $O | grep $TAG
