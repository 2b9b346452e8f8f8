set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_dist_gpu.py -q -k "fused and red_tma" > gpurun_out/pytest_redtma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_redtma.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 scripts/step_bench.py --layers 8 --tokens 8192 --rounds 4 > gpurun_out/step4.json 2> gpurun_out/step4.err
echo done
