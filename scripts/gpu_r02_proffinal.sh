# final per-pass ncu table of QAOA-30 (address-pattern counter-measures in)
cd $GRAFT_REPO_ROOT
T=/tmp/r02pf; mkdir -p $T
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pf2_build.log 2>&1
timeout 1500 ncu --profile-from-start off --set full --clock-control none -k regex:jit -c 12 \
  -o $T/qaoa30 python scripts/prof_passes.py qaoa 30 > gpurun_out/pf2_ncu_qaoa.log 2>&1
echo "rc=$?" >> gpurun_out/pf2_ncu_qaoa.log
ncu -i $T/qaoa30.ncu-rep --page raw --csv > gpurun_out/pf2_qaoa30_raw.csv 2>/dev/null
python scripts/prof_passes.py qaoa 30 --plan > gpurun_out/pf2_qaoa30_plan.txt 2>&1 || true
