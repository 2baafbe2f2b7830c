cd $GRAFT_REPO_ROOT
CMD="python bench.py --workload diag --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_diag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jit -s 2 -c 2 \
  -o gpurun_out/prof_diag $CMD > gpurun_out/ncu_diag_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_diag_full.log
