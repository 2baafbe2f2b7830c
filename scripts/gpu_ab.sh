cd $GRAFT_REPO_ROOT
for i in 1 2; do
for V in "QS_AB=default" "QS_BOOST_LOW=12 QS_WO_BUDGET=400" "QS_BOOST_LOW=12" "QS_WO_BUDGET=100"; do
  env $V timeout 300 python bench.py --workload qft --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > "gpurun_out/ab_${V// /_}_qft_$i.log" 2>&1
done; done
