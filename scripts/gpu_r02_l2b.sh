# f2 co-scheduled runs: parity, QFT-30 split sweep
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2b_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "l2_blocked or qft or rzz" > gpurun_out/l2b_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/l2b_pytest.txt
QS_L2_BLOCK=0 timeout 300 python bench.py --workload qft --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2b_qft_off.json 2> gpurun_out/l2b_qft_off.err
for sp in 1,1 2,1 1,2 3,2 2,3; do
  QS_L2_SPLIT=$sp timeout 300 python bench.py --workload qft --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2b_qft_$sp.json 2> gpurun_out/l2b_qft_$sp.err
done
timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/l2b_pytest2.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/l2b_pytest2.txt
