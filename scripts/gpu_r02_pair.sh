# chunk-pair dealing (QS_JIT_PAIR) A/B + parity with it
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pair_build.log 2>&1
QS_JIT_PAIR=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pair_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pair_pytest.txt
for wl in qaoa rand qft diag; do
  for P in 0 1; do
    QS_JIT_PAIR=$P QS_TIMING_DUMP=1 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pair_${wl}_$P.json 2> gpurun_out/pair_${wl}_$P.err
  done
done
