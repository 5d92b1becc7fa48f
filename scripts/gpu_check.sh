# One GPU round trip: smoke, GPU tests, K2 variant sweep, bench, launch list, ncu of K2.
# usage: bash scripts/gpu_check.sh <tag> [pytest -k expr]
set -x
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q ${2:+-k "$2"} 2>&1 | tail -15
timeout 600 python scripts/k2_sweep.py > gpurun_out/sweep_$TAG.jsonl 2> gpurun_out/sweep_$TAG.err; tail -2 gpurun_out/sweep_$TAG.err
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rgcsr_spmv -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log
ls gpurun_out
