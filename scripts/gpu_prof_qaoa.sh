cd $GRAFT_REPO_ROOT
CMD="python bench.py --workload qaoa --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_qaoa.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1_chunk -s 12 -c 5 \
  -o gpurun_out/prof_qaoa $CMD > gpurun_out/ncu_qaoa_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_qaoa_full.log
