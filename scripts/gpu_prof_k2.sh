# ncu --set full with source of the QFT-30 write-only pass (K2), after a clean run
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2 -s 1 -c 1 \
  -o gpurun_out/prof_k2 $CMD1 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
