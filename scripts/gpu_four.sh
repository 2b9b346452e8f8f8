set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 scripts/step_bench.py --layers 8 --tokens 8192 > gpurun_out/step4.json 2> gpurun_out/step4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29693 scripts/reconfig_check.py bench 2 0 4 > gpurun_out/reconfig_bench4.json 2> gpurun_out/reconfig_bench4.err
echo done
