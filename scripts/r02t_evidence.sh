# Final round-2 evidence on one B200 (session 3): smoke, 3 bench lines, the
# reference arm, the bench launch list, ncu --set full of the headline kernel.
# usage: bash scripts/r02t_evidence.sh <tag>
TAG=${1:-r02t}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; tail -1 $O/smoke_$TAG.log
for i in 1 2 3; do
  timeout 900 python bench.py > $O/bench_${TAG}_$i.json 2> $O/bench_${TAG}_$i.err; tail -c 200 $O/bench_${TAG}_$i.json; echo
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2>&1; tail -c 200 $O/bench_ref_$TAG.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live > /dev/null 2>&1; echo launches $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rgcsr_spmv -s 3 -c 1 -o $O/prof_headline_$TAG python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live --no-powerlaw > $O/ncu_headline_$TAG.log 2>&1; tail -1 $O/ncu_headline_$TAG.log
ls $O | grep $TAG
