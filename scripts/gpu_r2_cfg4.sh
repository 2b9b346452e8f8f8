# BASELINE configs[4] refresh: 8B-shaped TP4->TP3/TP2 reconfiguration (1 GPU sweep) and the
# multi-GPU failure reconfiguration bench at N=1/2/4, final code
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python scripts/sweep.py > gpurun_out/cfg4_sweep_n1.json 2> gpurun_out/cfg4_sweep_n1.err
for n in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2993$n scripts/reconfig_check.py bench 4 1 2 > gpurun_out/cfg4_reconfig_n$n.json 2> gpurun_out/cfg4_reconfig_n$n.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29934 scripts/reconfig_check.py bench 2 0 4 > gpurun_out/cfg4_reconfig_n4.json 2> gpurun_out/cfg4_reconfig_n4.err
echo done
