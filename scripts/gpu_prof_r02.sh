# round 2: per-pass launch lists + ncu --set full of the QAOA-30 / rand-30
# circuits.  Big reports stay in /tmp on the box; CSV summaries come back.
cd $GRAFT_REPO_ROOT
T=/tmp/r02prof; mkdir -p $T
for wl in qaoa rand; do
  timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02p_bench_$wl.json 2> gpurun_out/r02p_bench_$wl.err
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02p_launches_$wl.csv python scripts/prof_passes.py $wl 30 > gpurun_out/r02p_ll_$wl.log 2>&1
done
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jit -c 12 \
  -o $T/r02p_qaoa30 python scripts/prof_passes.py qaoa 30 > gpurun_out/r02p_ncu_qaoa.log 2>&1
echo "qaoa rc=$?" >> gpurun_out/r02p_ncu_qaoa.log
timeout 2400 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jit -c 40 \
  -o $T/r02p_rand30 python scripts/prof_passes.py rand 30 > gpurun_out/r02p_ncu_rand.log 2>&1
echo "rand rc=$?" >> gpurun_out/r02p_ncu_rand.log
for r in qaoa30 rand30; do
  ncu -i $T/r02p_$r.ncu-rep --page raw --csv > gpurun_out/r02p_${r}_raw.csv 2>/dev/null
  python scripts/ncu_summary.py $T/r02p_$r.ncu-rep > gpurun_out/r02p_${r}_summary.txt 2>&1
  ls -la $T/r02p_$r.ncu-rep >> gpurun_out/r02p_sizes.txt
  sz=$(stat -c %s $T/r02p_$r.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -lt 20000000 ]; then cp $T/r02p_$r.ncu-rep gpurun_out/; fi
done
