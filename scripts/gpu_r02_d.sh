# round 2, call D: ring-depth / group-count A/B and the coalesced write-only
# expansion, QAOA-30 / rand-30 / QFT-30; parity of the variants at n = 24
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1
run() { tag=$1; shift; for wl in qaoa rand qft; do
  env "$@" timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/r02d_${tag}_$wl.json 2> gpurun_out/r02d_${tag}_$wl.err; done; }
run base QS_X=0
run noxsm QS_JIT_NOXSM=1
run g1nb2 QS_JIT_GROUPS=1 QS_JIT_NB=2
run g1nb3 QS_JIT_GROUPS=1 QS_JIT_NB=3
run g2nb3 QS_JIT_GROUPS=2 QS_JIT_NB=3
QS_JIT_GROUPS=1 QS_JIT_NB=3 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/r02d_pytest_g1nb3.txt 2>&1
echo "rc=$?" >> gpurun_out/r02d_pytest_g1nb3.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/r02d_pytest_default.txt 2>&1
echo "rc=$?" >> gpurun_out/r02d_pytest_default.txt
