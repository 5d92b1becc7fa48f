# Refresh the round's evidence on one B200: smoke, the GPU suite, the bench
# line, the ncu launch list + headline capture, the SURVEY 8d records, the
# distributed path at P=1 (+ 2 ranks sharing the GPU), the K2 sweep.
# usage: bash scripts/round_end.sh <tag>
TAG=${1:-final}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; tail -1 $O/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_$TAG.log 2>&1; tail -1 $O/pytest_$TAG.log
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; tail -c 300 $O/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2>&1; tail -c 300 $O/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rgcsr_spmv -s 3 -c 1 -o $O/prof_$TAG python bench.py --steps 5 --warmup 3 --cpu-reps 1 --no-traffic-live > $O/ncu_$TAG.log 2>&1; tail -1 $O/ncu_$TAG.log
timeout 1200 python scripts/records.py --out $O/records_$TAG.jsonl > $O/records_$TAG.log 2>&1; tail -2 $O/records_$TAG.log
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import records_ncu as r; print(r.METRICS)")
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file $O/rec_ncu_$TAG.csv -k regex:"rgcsr_spmv|hybrid_spmv|csr_spmv|dot_partials" python scripts/records_ncu.py run > $O/rec_ncu_$TAG.log 2>&1
python scripts/records_ncu.py merge $O/rec_ncu_$TAG.csv $O/records_$TAG.jsonl
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29541 bench.py --distributed --workload 7pt-512 --steps 50 --warmup 5 > $O/dist1_fused_$TAG.json 2> $O/dist1_fused_$TAG.err; tail -c 300 $O/dist1_fused_$TAG.json
SPMVK_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29542 bench.py --gpus 2 --steps 50 --warmup 5 > $O/dist2_shared_$TAG.json 2> $O/dist2_shared_$TAG.err; tail -c 300 $O/dist2_shared_$TAG.json
timeout 600 python scripts/k2_sweep.py > $O/sweep_$TAG.jsonl 2> $O/sweep_$TAG.err
ls $O | grep $TAG
