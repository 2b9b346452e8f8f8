# sync kernel variant per size at N=2 (CUDA-graph steps)
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
for v in 1 2 3; do
NTP_SYNC_KERNEL=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2988$v scripts/sweep.py --sync-only > gpurun_out/z_sweep_k$v.json 2> gpurun_out/z_sweep_k$v.err
done
echo done
