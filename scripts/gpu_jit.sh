# GPU parity tests + bench (qft/rzz/diag/qaoa) + ncu of the specialised K1 kernel + launch list
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
for w in rzz diag qaoa; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$w.log 2>&1; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qs_k[123]_ -s 2 -c 2 \
  -o gpurun_out/prof_k1jit $CMD > gpurun_out/ncu.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
timeout 600 python scripts/kbench.py > gpurun_out/kbench.log 2>&1
