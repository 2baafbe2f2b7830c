cd $GRAFT_REPO_ROOT
timeout 1500 python scripts/roster.py --n 31 > gpurun_out/roster.jsonl 2> gpurun_out/roster.err
echo "roster rc=$?" >> gpurun_out/roster.err
