set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_fused_gpu.py -x -q > gpurun_out/pytest_splitk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_splitk.log
timeout 600 python scripts/gemm_bench.py > gpurun_out/gemm_splitk.json 2> gpurun_out/gemm_splitk.err; echo "rc=$?" >> gpurun_out/gemm_splitk.err
timeout 200 python scripts/splitk_trace.py 4779 fwd1 > gpurun_out/trace_f.json 2>&1
echo done
