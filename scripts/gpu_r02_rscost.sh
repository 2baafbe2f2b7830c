# cost model with row scaling: parity + QAOA/rand
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rc_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rc_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/rc_pytest.txt
for wl in qaoa rand diag qft; do
  timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rc_${wl}.json 2>/dev/null
done
