# round 2, call I: new GPU tests; ncu of rand-30 after unit-scaled ops
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/r02i_pytest_fullsize.txt 2>&1
echo "rc=$?" >> gpurun_out/r02i_pytest_fullsize.txt
T=/tmp/r02i; mkdir -p $T
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k1_chunk -c 8 \
  -o $T/rand8 python scripts/prof_passes.py rand 30 > gpurun_out/r02i_ncu_rand.log 2>&1
ncu -i $T/rand8.ncu-rep --page raw --csv > gpurun_out/r02i_rand_raw.csv 2>/dev/null
for i in 1 4; do ncu -i $T/rand8.ncu-rep --page source --csv --print-source sass -s $i -c 1 > gpurun_out/r02i_rand_src$i.csv 2>/dev/null; done
