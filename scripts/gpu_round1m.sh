set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q > gpurun_out/pytest_dist6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist6.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29414 bench.py --gpus 2 > gpurun_out/bench_n2c.json 2> gpurun_out/bench_n2c.err; echo "rc=$?" >> gpurun_out/bench_n2c.err
echo done
