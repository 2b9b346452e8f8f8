set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q -x > gpurun_out/pytest_dist5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist5.log
echo done
