set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_signals_gpu.py tests/test_fused_gpu.py -q > gpurun_out/pytest_sig.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sig.log
echo done
