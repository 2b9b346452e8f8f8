# BN=224 pair tiles: GEMM parity (all tile paths), bounds, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_linear_gpu.py tests/test_bounds_gpu.py tests/test_fused_gpu.py tests/test_dropin_gpu.py -q > gpurun_out/o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/o_tests.log
timeout 900 python scripts/gemm_bench.py > gpurun_out/o_gemm_bench.json 2> gpurun_out/o_gemm_bench.err
echo done
