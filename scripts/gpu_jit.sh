# GPU parity tests + bench (qft/rzz/diag) + ncu of the specialised K1 kernel
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
for w in rzz diag; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$w.log 2>&1; done
python -c "import paper_2604_12256_b200 as qs; print(qs.jit_info())" >> gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qs_k1_chunk_jit -s 2 -c 2 \
  -o gpurun_out/prof_k1jit $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
