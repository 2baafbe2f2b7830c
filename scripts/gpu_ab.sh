cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
for V in "QS_JIT_NOTENSOR=1" "QS_TENSOR=1"; do
  env $V timeout 300 python bench.py --workload qaoa --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > "gpurun_out/ab_${V}_qaoa_$i.log" 2>&1
  env $V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ablaunch_${V}_$i.csv python bench.py --workload qaoa --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done; done
