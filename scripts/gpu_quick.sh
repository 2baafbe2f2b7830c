# GPU parity tests + kernel calibration + benches (no ncu)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/kbench.py > gpurun_out/kbench.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench.log 2>&1
for w in rzz diag qaoa; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$w.log 2>&1; done
