# round 2, call G: multi-copy tensor TMA A/B (QS_JIT_TENSOR_COPIES) on QAOA-30
# and rand-30, and parity of the multi-copy loads
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g_build.log 2>&1
for mc in 1 32 64 128 256; do
  for wl in qaoa rand; do
    QS_JIT_TENSOR_COPIES=$mc timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/r02g_tc${mc}_$wl.json 2> gpurun_out/r02g_tc${mc}_$wl.err
  done
done
QS_JIT_TENSOR_COPIES=256 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/r02g_pytest_tc256.txt 2>&1
echo "rc=$?" >> gpurun_out/r02g_pytest_tc256.txt
