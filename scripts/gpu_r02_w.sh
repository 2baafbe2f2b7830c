cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02w_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02w_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02w_pytest_gpu.txt
for wl in qft rzz diag qaoa rand; do
  QS_PLAN_TIMING=1 timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02w_$wl.json 2> gpurun_out/r02w_$wl.err
done
