# per-launch timings (QS_TIMING_DUMP) of one circuit of each workload, 1 GPU
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1
for wl in qft diag qaoa rand rzz; do
  QS_TIMING_DUMP=1 timeout 600 python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02j_$wl.json 2> gpurun_out/r02j_$wl.err
done
