# one-qubit row scaling (RX/RY -> unit diagonal + pass scale): parity + A/B
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rs_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rs_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/rs_pytest.txt
for wl in qaoa rand; do
  QS_NO_ROWSCALE=1 timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rs_${wl}_off.json 2>/dev/null
  timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rs_${wl}_on.json 2>/dev/null
done
