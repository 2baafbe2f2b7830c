# round 2, call H: hoisted-gather grid (148 -> 144 CTAs) A/B on the write-only
# passes; GPU tests with the final defaults
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1
for x in 1 0; do
  for wl in qft rzz diag qaoa; do
    QS_JIT_XHGRID=$x timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/r02h_xh${x}_$wl.json 2> gpurun_out/r02h_xh${x}_$wl.err
  done
done
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02h_pytest_gpu.txt
