set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --steps 400 --warmup 5 > gpurun_out/bench3_n1.json 2> gpurun_out/bench3_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29411 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench3_n2.json 2> gpurun_out/bench3_n2.err
echo done
