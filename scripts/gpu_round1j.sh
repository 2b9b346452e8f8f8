set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_linear_gpu.py -q -x > gpurun_out/pytest_linear3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_linear3.log
timeout 300 python scripts/gemm_bench.py 8192 > gpurun_out/gemm_bench3.json 2> gpurun_out/gemm_bench3.err
echo done
