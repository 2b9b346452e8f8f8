# bench N=2 / N=1 lines after dropping NVML, small probe
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/h_bench_c2_n2.json 2> gpurun_out/h_bench_c2_n2.err
timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 > gpurun_out/h_bench_c1_n2.json 2> gpurun_out/h_bench_c1_n2.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --workload llama3-8b-shaped --no-e2e > gpurun_out/h_bench_c4_n2.json 2> gpurun_out/h_bench_c4_n2.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/h_bench_c2_n1.json 2> gpurun_out/h_bench_c2_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29770 scripts/sweep.py --sync-only > gpurun_out/h_sweep_n2.json 2> gpurun_out/h_sweep_n2.err
echo done
