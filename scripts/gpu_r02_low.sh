# forced low run of chunk positions (QS_PLAN_LOW 3 vs 4): QAOA / rand
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/low_build.log 2>&1
for wl in qaoa rand; do
  for L in 3 4; do
    QS_PLAN_LOW=$L QS_TIMING_DUMP=1 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/low_${wl}_$L.json 2> gpurun_out/low_${wl}_$L.err
  done
done
