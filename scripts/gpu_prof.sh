# ncu --set full of one K2 configuration per argument "case:prec:variant[:format]"
set -x
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read kind n G prec variant fmt <<< "$spec"
  tag="${kind}pt${n}_g${G}_p${prec}_${variant}_${fmt:-rgcsr}"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rgcsr_spmv|hybrid_spmv" -s 2 -c 1 \
      -o gpurun_out/prof_$tag python scripts/prof_k2.py --case $kind:$n:$G --prec $prec --variant $variant --format ${fmt:-rgcsr} > gpurun_out/ncu_$tag.log 2>&1
  tail -1 gpurun_out/ncu_$tag.log
done
