# A/B: resident-CTA target of write-only passes (QS_JIT_WO_MINB), QFT-30 and RZZ-30 (same box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0"
for w in qft rzz diag; do
  for m in def 1; do
    if [ $m = def ]; then timeout 300 $B --workload $w > gpurun_out/ab_${w}_$m.log 2>&1
    else QS_JIT_WO_MINB=$m timeout 300 $B --workload $w > gpurun_out/ab_${w}_$m.log 2>&1; fi
  done
done
QS_JIT_WO_MINB=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "parity or qft or rzz" > gpurun_out/ab_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ab_pytest.log
