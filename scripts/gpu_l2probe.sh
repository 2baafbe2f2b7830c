cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_probe scripts/dev/l2_probe.cu && timeout 300 /tmp/l2_probe > gpurun_out/l2_probe.jsonl 2>&1
echo "rc=$?" >> gpurun_out/l2_probe.jsonl
