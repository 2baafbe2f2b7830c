# NaN-poisoned consumed buffers + ring-phase asserts (QS_JIT_CHECK) on the full-size parity tests, final code
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ck2_build.log 2>&1
QS_JIT_CHECK=1 QS_JIT_CACHE=/tmp/ck_cache timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/ck2_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/ck2_pytest.txt
