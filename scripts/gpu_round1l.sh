set -x
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 scripts/dp_check.py 2 2 1 bf16 2 > gpurun_out/dp_bf16.out 2> gpurun_out/dp_bf16.err
echo done
