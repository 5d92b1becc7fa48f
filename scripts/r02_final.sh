# Round-2 final evidence on one B200: smoke, GPU suite, 3 bench lines + the
# reference arm, bench launch list, ncu of the headline kernel, the SURVEY 8d
# records with ncu counters, memcheck over the sanitize pass.
# usage: bash scripts/r02_final.sh <tag> [skip-tests]
TAG=${1:-r02f}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; tail -1 $O/smoke_$TAG.log
if [ -z "$2" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_$TAG.log 2>&1; tail -2 $O/pytest_$TAG.log
fi
for i in 1 2 3; do
  timeout 900 python bench.py > $O/bench_${TAG}_$i.json 2> $O/bench_${TAG}_$i.err; tail -c 200 $O/bench_${TAG}_$i.json; echo
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2>&1; tail -c 200 $O/bench_ref_$TAG.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rgcsr_spmv -s 3 -c 1 -o $O/prof_headline_$TAG python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live --no-powerlaw > $O/ncu_headline_$TAG.log 2>&1; tail -1 $O/ncu_headline_$TAG.log
timeout 1500 python scripts/records.py --out $O/records_$TAG.jsonl > $O/records_$TAG.log 2>&1; tail -2 $O/records_$TAG.log
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import records_ncu as r; print(r.METRICS)")
timeout 1800 ncu --metrics $M --clock-control none --csv --log-file $O/rec_ncu_$TAG.csv -k regex:"rgcsr_spmv|hybrid_spmv|hybrid_ell_vec|csr_spmv|dot_partials" python scripts/records_ncu.py run > $O/rec_ncu_$TAG.log 2>&1
python scripts/records_ncu.py merge $O/rec_ncu_$TAG.csv $O/records_$TAG.jsonl
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize.py > $O/san_${TAG}_memcheck.log 2>&1; tail -2 $O/san_${TAG}_memcheck.log
ls $O | grep $TAG
