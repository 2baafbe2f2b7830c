# shape-table kernel with column groups: parity + A/B + launch list
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tab2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/tab2_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/tab2_pytest.txt
for wl in qft diag qaoa rand rzz; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tab2_${wl}.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tab2_launches_qft.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tab2_ncu.log 2>&1
