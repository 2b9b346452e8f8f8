set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q -k fused > gpurun_out/pytest_fused_dist.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fused_dist.log
echo done
