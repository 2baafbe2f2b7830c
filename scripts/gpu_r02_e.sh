# round 2, call E: unit-scaled ops + quarter-turn diagonals + 2-group
# write-only passes: GPU tests (default and with QS_JIT_CHECK poisoning),
# bench of every workload, write-only budget A/B on QFT-30
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02e_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02e_pytest_gpu.txt
QS_JIT_CHECK=1 timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/r02e_pytest_check.txt 2>&1
echo "rc=$?" >> gpurun_out/r02e_pytest_check.txt
for wl in qft rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02e_$wl.json 2> gpurun_out/r02e_$wl.err
done
for b in 32 36 40 44; do
  QS_WO_BUDGET=$b timeout 600 python bench.py --workload qft --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02e_wob$b.json 2>&1
done
QS_JIT_NOQUARTER=1 timeout 600 python bench.py --workload rand --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02e_rand_noquarter.json 2>&1
