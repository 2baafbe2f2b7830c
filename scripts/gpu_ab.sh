cd $GRAFT_REPO_ROOT
for i in 1 2; do
for V in 0 1 2; do
  for w in qft qaoa diag; do
  QS_JIT_DIAGPROD=$V timeout 300 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > "gpurun_out/ab_${V}_${w}_$i.log" 2>&1
  done
done; done
