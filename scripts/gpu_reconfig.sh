set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_dist_gpu.py -q -k reconfig > gpurun_out/pytest_reconfig.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_reconfig.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 scripts/reconfig_check.py bench 4 1 2 > gpurun_out/reconfig_bench2.json 2> gpurun_out/reconfig_bench2.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29672 scripts/reconfig_check.py bench 4 1 2 > gpurun_out/reconfig_bench1.json 2> gpurun_out/reconfig_bench1.err
echo done
