# round 2, first box: full-size parity, bench N=1 (C2 --check, C1), N=2 via re-exec, NVML probe
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
timeout 600 python -m pytest tests/test_fullsize_gpu.py -x -q > gpurun_out/a_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/a_fullsize.log
timeout 300 python scripts/nvml_nvlink_probe.py > gpurun_out/a_nvml.json 2> gpurun_out/a_nvml.err
timeout 600 python bench.py --steps 20 --warmup 5 --check > gpurun_out/a_bench_c2.json 2> gpurun_out/a_bench_c2.err
timeout 600 python bench.py --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 --check > gpurun_out/a_bench_c1.json 2> gpurun_out/a_bench_c1.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/a_bench_n2.json 2> gpurun_out/a_bench_n2.err
timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 --no-e2e > gpurun_out/a_bench_c1_n2.json 2> gpurun_out/a_bench_c1_n2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/a_ref_c2.json 2> gpurun_out/a_ref_c2.err
echo done
