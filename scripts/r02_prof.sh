#!/bin/bash
# ncu captures for round 2: one launch per configuration (after 2 warm-up
# launches), --set full.  Args: "kind:n:G:prec:variant:format[:hvariant[:reorder]]"
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read kind n G prec variant fmt hv ro <<< "$spec"
  tag="r02_${kind}pt${n}_g${G}_p${prec}_${variant}_${fmt}_${hv:-auto}${ro:+_r}"
  extra=""; [ -n "$ro" ] && extra="--reorder"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"rgcsr_spmv|hybrid_spmv|hybrid_heavy" -s 2 -c 2 -o gpurun_out/prof_$tag \
      python scripts/prof_k2.py --case $kind:$n:$G --prec $prec --variant $variant \
      --format $fmt --hvariant ${hv:-auto} $extra > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
done
