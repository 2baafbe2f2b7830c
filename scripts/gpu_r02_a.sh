# round 2, call A: GPU tests (incl. the full-size parity file), smoke, QFT-30
# bench line, then per-pass launch lists + ncu --set full of QAOA-30/rand-30
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a_build.log 2>&1
nproc > gpurun_out/r02a_host.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/r02a_host.txt; free -g >> gpurun_out/r02a_host.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/r02a_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a_pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/r02a_smoke.txt
timeout 900 python bench.py > gpurun_out/r02a_bench_qft.json 2> gpurun_out/r02a_bench_qft.err
bash scripts/gpu_prof_r02.sh
du -sh gpurun_out >> gpurun_out/r02p_sizes.txt
