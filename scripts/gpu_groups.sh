cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in qft rzz qaoa diag; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > "gpurun_out/bench_$w.log" 2>&1
done
for w in qaoa diag qft; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$w.log 2>&1
done
