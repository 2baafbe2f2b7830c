# L2 prefetch per refill engine: A/B on QAOA / rand / QFT / diag, parity with it on
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pf_build.log 2>&1
QS_JIT_L2PF=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pf_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pf_pytest.txt
for wl in qaoa rand qft diag; do
  for pf in 0 1 2; do
    QS_JIT_L2PF=$pf timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pf_${wl}_$pf.json 2> gpurun_out/pf_${wl}_$pf.err
  done
done
