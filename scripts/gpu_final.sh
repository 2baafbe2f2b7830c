# parity + smoke + default bench (cpu baseline, e2e) + reference arm + all workloads + launch list + full ncu of the QFT-30 passes
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for w in rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$w.log 2>&1
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jit -s 2 -c 2 \
  -o gpurun_out/prof_qft $CMD1 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
