# host-side timeline of a QFT-30 / RZZ-30 step (QS_PLAN_TIMING) + the sweep test
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1
for wl in qft rzz; do
  QS_PLAN_TIMING=1 timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02u_$wl.json 2> gpurun_out/r02u_$wl.err
done
timeout 900 python -m pytest tests/test_gpu_sweep.py -q > gpurun_out/r02u_sweep.txt 2>&1
