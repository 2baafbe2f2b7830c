# f2 co-scheduled runs: parity (deadlock-free lag), QFT-30 diagnostics
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2e_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "l2_blocked or qft" > gpurun_out/l2e_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/l2e_pytest.txt
run() { timeout 120 python bench.py --workload qft --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2e_qft_$1.json 2> gpurun_out/l2e_qft_$1.err; }
QS_L2_SPLIT=1,2 run base12
QS_L2_SPLIT=1,1 run base11
QS_L2_SPLIT=1,2 QS_RUN_NOPFENCE=1 run nopf12
QS_L2_SPLIT=1,2 QS_RUN_SLEEP=0 run nosleep12
QS_L2_SPLIT=1,2 QS_L2_LAG=8 run lag8
QS_L2_SPLIT=1,2 QS_RUN_PROF=1 run prof12
QS_L2_SPLIT=1,1 QS_RUN_PROF=1 run prof11
