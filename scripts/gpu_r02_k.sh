# ncu of QAOA-30's first (write-only, multi-layout) pass
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02k_build.log 2>&1
T=/tmp/r02k; mkdir -p $T
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k1_chunk -c 1 \
  -o $T/qaoa_wo python scripts/prof_passes.py qaoa 30 > gpurun_out/r02k_ncu.log 2>&1
ncu -i $T/qaoa_wo.ncu-rep --page raw --csv > gpurun_out/r02k_qaoa_wo_raw.csv 2>/dev/null
ncu -i $T/qaoa_wo.ncu-rep --page source --csv --print-source sass > gpurun_out/r02k_qaoa_wo_src.csv 2>/dev/null
QS_JIT_DUMP=gpurun_out python -c "
import sys; sys.path.insert(0,'.')
import bench, paper_2604_12256_b200 as qs
g=bench.make_circuit('qaoa',30)
qs.plan_json(30,g,basis=bench.BASIS_X%(1<<30),detail=2)
" > /dev/null 2>&1
mkdir -p gpurun_out/r02k_src; mv gpurun_out/*_qs_k*_jit.cu gpurun_out/r02k_src/ 2>/dev/null
