set -x
mkdir -p gpurun_out
timeout 300 python scripts/gemm_bench.py 8192 > gpurun_out/gemm_bench.json 2> gpurun_out/gemm_bench.err
timeout 600 python scripts/sweep.py --reconfig-layers 32 > gpurun_out/sweep.json 2> gpurun_out/sweep.err
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plan_kernel_bulk -s 3 -c 1 -o gpurun_out/prof_bulk python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bulk.log 2>&1
timeout 300 python scripts/gemm_bench.py 8192 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 5 -c 1 -o gpurun_out/prof_gemm python scripts/gemm_bench.py 8192 > gpurun_out/ncu_gemm.log 2>&1
echo done
