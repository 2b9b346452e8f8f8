# min-chunks experiment: N=2 sweep at 0 / 1184 / 2368 / 4736 minimum chunks per plan
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
for mc in 0 1184 2368 4736; do
NTP_MIN_CHUNKS=$mc timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2985$((mc % 7)) scripts/sweep.py --sync-only > gpurun_out/t_sweep_mc$mc.json 2> gpurun_out/t_sweep_mc$mc.err
done
echo done
