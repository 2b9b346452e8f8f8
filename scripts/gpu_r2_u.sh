# after the min-chunks default: whole GPU suite (4 GPUs), sweeps N=2/4, bench lines N=1/2/4 (C1, C2)
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/u_bench_c2_n1.json 2> gpurun_out/u_bench_c2_n1.err
timeout 600 python bench.py --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 > gpurun_out/u_bench_c1_n1.json 2> gpurun_out/u_bench_c1_n1.err
for n in 2 4; do
timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/u_bench_c2_n$n.json 2> gpurun_out/u_bench_c2_n$n.err
timeout 600 python bench.py --gpus $n --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 > gpurun_out/u_bench_c1_n$n.json 2> gpurun_out/u_bench_c1_n$n.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2986$n scripts/sweep.py --sync-only > gpurun_out/u_sweep_n$n.json 2> gpurun_out/u_sweep_n$n.err
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/u_pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/u_pytest_gpu4.log
echo done
