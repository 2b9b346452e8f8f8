set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 scripts/step_bench.py --layers 8 --tokens 8192 --rounds 5 > gpurun_out/step4.json 2> gpurun_out/step4.err
echo done
