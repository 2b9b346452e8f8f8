# the N=8 placement (7 logical ranks + an idle one) as 8 processes on 4 GPUs (2 per GPU, gloo host group)
mkdir -p gpurun_out
for launch in three graph; do
SECONDS=0
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 2989${#launch} scripts/dist_check.py 4 3 bf16 2 $launch > gpurun_out/os_$launch.log 2>&1; echo "rc=$? seconds=$SECONDS" >> gpurun_out/os_$launch.log
done
echo done
