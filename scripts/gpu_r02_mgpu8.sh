# pull-pass load engine A/B (TMA bulk vs per-thread cp.async) at 4 GPUs
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02s_build.log 2>&1
for v in 0 1; do
  for wl in qaoa rand; do
    if [ $v = 1 ]; then E="QS_JIT_PULL_CPASYNC=1"; else E="QS_X=0"; fi
    env $E QS_TIMING_DUMP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29850 + v)) \
      bench.py --gpus 4 --steps 3 --warmup 3 --workload $wl --e2e-steps 0 > gpurun_out/r02s_${wl}_v$v.log 2> gpurun_out/r02s_${wl}_v$v.err
  done
done
