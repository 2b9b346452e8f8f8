# canary bounds tests, 1-GPU group/overlapped-step tests (vs oracle), 2-GPU overlapped step, signal latency
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_bounds_gpu.py -q > gpurun_out/j_bounds.log 2>&1; echo "rc=$?" >> gpurun_out/j_bounds.log
timeout 900 python -m pytest tests/test_dist_gpu.py -k "one_gpu or overlapped" -q > gpurun_out/j_dist.log 2>&1; echo "rc=$?" >> gpurun_out/j_dist.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29790 scripts/probes/signal_latency.py > gpurun_out/j_siglat.json 2> gpurun_out/j_siglat.err
echo done
