mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_dist_gpu.py -k "graph" -q > gpurun_out/x_tests.log 2>&1; echo "rc=$?" >> gpurun_out/x_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29870 scripts/sweep.py --sync-only > gpurun_out/x_sweep_n2.json 2> gpurun_out/x_sweep_n2.err
echo done
