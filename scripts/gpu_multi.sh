set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 600 python -m pytest tests/test_multi.py -q > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi.log
timeout 900 python -m pytest tests/test_dist_gpu.py -q -k "c3_shape" > gpurun_out/pytest_dp.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dp.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 scripts/dp_bench.py 3 2 1 10 1,8 > gpurun_out/dp_bench.json 2> gpurun_out/dp_bench.err
echo done
