# e2e A/B on one box: env settings of the host-span pipeline, fresh processes,
# spmvk_host_alloc buffers (scripts/e2e_timeline.py prints wall ms/step first)
for rep in 1 2 3; do
  for env in "SPMVK_PIPE_SPLIT=0" "SPMVK_PIPE_SPLIT=1"; do
    echo "$env: $(env $env E2E_ROWS=0 timeout 120 python scripts/e2e_timeline.py 2>/dev/null | grep wall)"
  done
done
