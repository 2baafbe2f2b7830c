# sub-state passes through the specialised kernels too (jit_min_qubits 18 vs 0 via QS_JIT=1)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/jm_build.log 2>&1
for wl in qft rzz diag qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/jm_${wl}_18.json 2>/dev/null
  QS_JIT=1 timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/jm_${wl}_0.json 2>/dev/null
done
