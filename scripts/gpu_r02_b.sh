# round 2, call B: QFT-30 write-only-pass A/B; full-state N=30 oracle parity
# of the five bench workloads; compute-sanitizer over the specialised kernels
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1
ab() { tag=$1; shift; env "$@" timeout 600 python bench.py --workload qft --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/r02b_${tag}_qft.json 2> gpurun_out/r02b_${tag}_qft.err; }
ab base QS_X=0
ab wog2 QS_JIT_WO_GROUPS=2
ab noxh QS_JIT_NOXH=1
ab wog2noxh QS_JIT_WO_GROUPS=2 QS_JIT_NOXH=1
ab wob40 QS_WO_BUDGET=40
ab wob56 QS_WO_BUDGET=56
ab wob40g2 QS_WO_BUDGET=40 QS_JIT_WO_GROUPS=2
ab wob56g2 QS_WO_BUDGET=56 QS_JIT_WO_GROUPS=2
free -g > gpurun_out/r02b_host.txt; nproc >> gpurun_out/r02b_host.txt
timeout 3000 python scripts/full_parity.py --n 30 --out gpurun_out/r02_full_parity_n30.jsonl > gpurun_out/r02b_full_parity.log 2>&1
echo "full parity rc=$?" >> gpurun_out/r02b_full_parity.log
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/r02b_sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02b_sanitize_$tool.txt
done
