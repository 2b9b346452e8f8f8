set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --steps 20 --warmup 3 --e2e-steps 8 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 scripts/dp_bench.py 3 2 1 10 8 > gpurun_out/dp_bench.json 2> gpurun_out/dp_bench.err
echo done
