set -x
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29412 scripts/nvlink_probe.py 1 > gpurun_out/nvprobe.json 2> gpurun_out/nvprobe.err
echo done
