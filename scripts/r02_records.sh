# SURVEY 8d records with ncu counters + sanitizer pass + one bench line.
# usage: bash scripts/r02_records.sh <tag>
TAG=${1:-r02g}
O=gpurun_out
mkdir -p $O
timeout 1800 python scripts/records.py --out $O/records_$TAG.jsonl > $O/records_$TAG.log 2>&1; tail -1 $O/records_$TAG.log
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import records_ncu as r; print(r.METRICS)")
timeout 1800 ncu --metrics $M --clock-control none --csv --log-file $O/rec_ncu_$TAG.csv -k regex:"rgcsr_spmv|hybrid_spmv|hybrid_ell_vec|csr_spmv|dot_partials" python scripts/records_ncu.py run > $O/rec_ncu_$TAG.log 2>&1
python scripts/records_ncu.py merge $O/rec_ncu_$TAG.csv $O/records_$TAG.jsonl
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py > $O/san_${TAG}_$tool.log 2>&1
  tail -2 $O/san_${TAG}_$tool.log
done
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; tail -c 300 $O/bench_$TAG.json
