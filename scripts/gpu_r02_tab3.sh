# small-table mapping: parity + QFT/RZZ/diag + launch list
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tab3_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/tab3_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/tab3_pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tab3_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/tab3_smoke.txt
for wl in qft rzz diag qaoa; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tab3_${wl}.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tab3_launches_qft.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tab3_ncu.log 2>&1
