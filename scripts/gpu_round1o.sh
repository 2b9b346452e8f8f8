set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused_gpu.py tests/test_linear_gpu.py -q -x > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fused.log
echo done
