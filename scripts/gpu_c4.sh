set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python bench.py --workload llama3-8b-shaped --steps 50 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c4_n1.json 2> gpurun_out/bench_c4_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --workload llama3-8b-shaped --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c4_n4.json 2> gpurun_out/bench_c4_n4.err
echo done
