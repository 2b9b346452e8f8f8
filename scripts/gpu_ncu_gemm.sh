set -x
mkdir -p gpurun_out
timeout 120 python scripts/gemm_one.py wgrad 4 > gpurun_out/g1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_wgrad python scripts/gemm_one.py wgrad 4 > gpurun_out/ncu_g1.log 2>&1
timeout 120 python scripts/gemm_one.py fwd1 4 > gpurun_out/g2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_fwd1 python scripts/gemm_one.py fwd1 4 > gpurun_out/ncu_g2.log 2>&1
echo done
