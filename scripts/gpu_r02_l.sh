# strict fusion A/B + GPU tests
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1
for t in 0 1; do
  for wl in qaoa rand qft diag; do
    if [ $t = 1 ]; then E="QS_FUSE_TIES=1"; else E="QS_X=0"; fi
    env $E QS_TIMING_DUMP=1 timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02l_t${t}_$wl.json 2> gpurun_out/r02l_t${t}_$wl.err
  done
done
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02l_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02l_pytest_gpu.txt
