# full-state N=30 oracle parity of the five bench workloads, final round-2 code
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fp2_build.log 2>&1
timeout 3000 python scripts/full_parity.py --n 30 --out gpurun_out/r02_full_parity_n30_final.jsonl > gpurun_out/fp2_full_parity.log 2>&1
echo "full parity rc=$?" >> gpurun_out/fp2_full_parity.log
