set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_linear_gpu.py -q -x > gpurun_out/pytest_linear.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_linear.log
timeout 300 python -m pytest tests/test_reconfig.py tests/test_cli.py -m gpu -q > gpurun_out/pytest_misc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_misc.log
echo done
