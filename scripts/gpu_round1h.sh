set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_linear_gpu.py tests/test_multi.py -q -x > gpurun_out/pytest_linear2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_linear2.log
timeout 300 python scripts/gemm_bench.py 8192 > gpurun_out/gemm_bench2.json 2> gpurun_out/gemm_bench2.err
echo done
