mkdir -p gpurun_out
python scripts/probes/pad_probe.py > gpurun_out/l_pad.log 2>&1
timeout 900 python -m pytest tests/test_bounds_gpu.py tests/test_linear_gpu.py tests/test_fused_gpu.py -q > gpurun_out/l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l_tests.log
timeout 600 python scripts/gemm_bench.py > gpurun_out/l_gemm_bench.json 2> gpurun_out/l_gemm_bench.err
echo done
