# round 2, call B: full-state N=30 oracle parity of the five bench workloads,
# and compute-sanitizer (racecheck/synccheck/memcheck) over the specialised
# kernels at n = 21-22
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1
free -g > gpurun_out/r02b_host.txt; nproc >> gpurun_out/r02b_host.txt
timeout 3000 python scripts/full_parity.py --n 30 --out gpurun_out/r02_full_parity_n30.jsonl > gpurun_out/r02b_full_parity.log 2>&1
echo "full parity rc=$?" >> gpurun_out/r02b_full_parity.log
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/r02b_sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02b_sanitize_$tool.txt
done
