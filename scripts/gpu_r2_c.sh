# round 2: GPU suite (2 GPUs, no -x), graph-step sweep at N=2, bench N=2 C1/C2
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c_pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/c_pytest_gpu2.log
timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 --no-e2e > gpurun_out/c_bench_c1_n2.json 2> gpurun_out/c_bench_c1_n2.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/c_bench_c2_n2.json 2> gpurun_out/c_bench_c2_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29720 scripts/sweep.py --sync-only > gpurun_out/c_sweep_n2.json 2> gpurun_out/c_sweep_n2.err
echo done
