# position-3 steering (QS_NO_STEER3) x chunk pairs on slow-pattern passes (QS_JIT_PAIR=0 vs default)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/steer_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/steer_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/steer_pytest.txt
for wl in qaoa rand; do
  QS_NO_STEER3=1 QS_JIT_PAIR=0 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/steer_${wl}_base.json 2>/dev/null
  QS_JIT_PAIR=0 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/steer_${wl}_s3.json 2>/dev/null
  timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/steer_${wl}_s3pair.json 2>/dev/null
  QS_NO_STEER3=1 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/steer_${wl}_pair.json 2>/dev/null
done
for wl in qft diag rzz; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/steer_${wl}_s3pair.json 2>/dev/null
done
