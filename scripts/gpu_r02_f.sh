# round 2, call F: GPU tests + smoke + every workload's bench line (QFT with
# the full contract), after the budget-candidate planner change
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02f_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f_pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02f_bench_qft.json 2> gpurun_out/r02f_bench_qft.err
for wl in rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02f_$wl.json 2> gpurun_out/r02f_$wl.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_reference.json 2> gpurun_out/r02f_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_qft.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02f_ncu_ll.log 2>&1
T=/tmp/r02f; mkdir -p $T
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jit -c 2 \
  -o $T/qft30 python scripts/prof_passes.py qft 30 > gpurun_out/r02f_ncu_qft.log 2>&1
ncu -i $T/qft30.ncu-rep --page raw --csv > gpurun_out/r02f_qft30_raw.csv 2>/dev/null
python scripts/ncu_summary.py $T/qft30.ncu-rep > gpurun_out/r02f_qft30_summary.txt 2>&1
for i in 0 1; do ncu -i $T/qft30.ncu-rep --page source --csv --print-source sass -s $i -c 1 > gpurun_out/r02f_qft_src$i.csv 2>/dev/null; done
