cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python scripts/roster.py --n 31 > gpurun_out/roster.jsonl 2> gpurun_out/roster.err
echo "roster rc=$?" >> gpurun_out/roster.err
