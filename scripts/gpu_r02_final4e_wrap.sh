# final 4-GPU run + the new one-GPU parity test
cd $GRAFT_REPO_ROOT
bash scripts/gpu_r02_final4e.sh
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "special_angles or qaoa or supremacy" > gpurun_out/r02f11_pytest_special.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f11_pytest_special.txt
