set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_reconfig.py tests/test_cli.py -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29411 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench4_n2.json 2> gpurun_out/bench4_n2.err
echo done
