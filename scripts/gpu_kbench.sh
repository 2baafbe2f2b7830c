cd $GRAFT_REPO_ROOT
timeout 900 python scripts/kbench.py > gpurun_out/kbench.log 2>&1
QS_JIT_GROUPS=1 timeout 900 python scripts/kbench.py > gpurun_out/kbench_g1.log 2>&1
