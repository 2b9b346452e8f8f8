set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 900 python -m pytest tests/test_dist_gpu.py -q > gpurun_out/pytest_dist4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29413 bench.py --gpus 4 --steps 100 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29414 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench_n2b.json 2> gpurun_out/bench_n2b.err
echo done
