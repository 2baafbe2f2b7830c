cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
for V in "QS_JIT_NOXH=1" "QS_XH=1"; do
  for w in qft diag rzz; do
  env $V timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > "gpurun_out/ab_${V}_${w}_$i.log" 2>&1
  done
done; done
