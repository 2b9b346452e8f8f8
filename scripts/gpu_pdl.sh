set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_fused_gpu.py -x -q > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pdl.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 scripts/step_bench.py --layers 8 --tokens 8192 --rounds 3 > gpurun_out/step4.json 2> gpurun_out/step4.err
echo done
