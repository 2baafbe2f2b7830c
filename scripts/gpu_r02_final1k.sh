# round 2 final single-GPU verification: tests, smoke, driver-style bench
# (QFT-30 full contract), the other workloads, the reference arm, launch list
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f17_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02f17_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f17_pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f17_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/r02f17_smoke.txt
timeout 900 python bench.py > gpurun_out/r02f17_bench_qft.json 2> gpurun_out/r02f17_bench_qft.err
for wl in rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02f17_$wl.json 2> gpurun_out/r02f17_$wl.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f17_reference.json 2> gpurun_out/r02f17_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f17_launches_qft.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02f17_ncu_ll.log 2>&1
