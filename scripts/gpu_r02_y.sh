# async accumulate mode: full GPU suite, 5 workloads
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02y2_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02y2_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02y2_pytest_gpu.txt
for wl in qft rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02y2_$wl.json 2> gpurun_out/r02y2_$wl.err
done
