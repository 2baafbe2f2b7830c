cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02v_build.log 2>&1
for wl in qft rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02v_$wl.json 2> gpurun_out/r02v_$wl.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "launch_count or qft30 or bench_workloads" > gpurun_out/r02v_pytest.txt 2>&1
