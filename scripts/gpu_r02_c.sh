# round 2, call C: L2-prefetch A/B on QAOA-30 / rand-30 / QFT-30, and
# source-level stall attribution of QAOA-30's first two read passes
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1
for pf in 0 2 4 8; do
  for wl in qaoa rand qft; do
    QS_JIT_L2PF=$pf timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/r02c_pf${pf}_$wl.json 2> gpurun_out/r02c_pf${pf}_$wl.err
  done
done
T=/tmp/r02c; mkdir -p $T
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k1_chunk -c 3 \
  -o $T/qaoa3 python scripts/prof_passes.py qaoa 30 > gpurun_out/r02c_ncu_qaoa.log 2>&1
for i in 0 1 2; do
  ncu -i $T/qaoa3.ncu-rep --page source --csv --print-source sass -s $i -c 1 > gpurun_out/r02c_qaoa_src$i.csv 2> gpurun_out/r02c_src$i.err
done
ls -la $T >> gpurun_out/r02c_ncu_qaoa.log
