cd $GRAFT_REPO_ROOT
for i in 1 2; do
for V in "QS_NO_LOW_STEER=1" "QS_STEER=1"; do
  for w in qaoa rand; do
  env $V timeout 300 python bench.py --workload $w --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 0 > "gpurun_out/ab_${V}_${w}_$i.log" 2>&1
  done
done; done
