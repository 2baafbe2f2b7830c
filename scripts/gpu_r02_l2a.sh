# f2 first GPU check: L2-blocked parity tests, QFT-30 wave-size sweep
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2a_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/l2a_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/l2a_pytest.txt
for wb in 0 20 21 22 23 24; do
  QS_L2_BLOCK=$wb timeout 300 python bench.py --workload qft --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2a_qft_$wb.json 2> gpurun_out/l2a_qft_$wb.err
done
for wl in qaoa rand; do
  for wb in 0 22; do
    QS_L2_BLOCK=$wb timeout 300 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/l2a_${wl}_$wb.json 2> gpurun_out/l2a_${wl}_$wb.err
  done
done
