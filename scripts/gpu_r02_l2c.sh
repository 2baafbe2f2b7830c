# f2 co-scheduled runs with backpressure: parity, QFT-30 split x lag sweep
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2c_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "l2_blocked or qft" > gpurun_out/l2c_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/l2c_pytest.txt
for sp in 1,1 1,2 2,3; do
  for lag in 4 16 48; do
    QS_L2_LAG=$lag QS_L2_SPLIT=$sp timeout 300 python bench.py --workload qft --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2c_qft_${sp}_$lag.json 2> gpurun_out/l2c_qft_${sp}_$lag.err
  done
done
