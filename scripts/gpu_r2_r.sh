mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_dist_gpu.py -k "row_parallel or prescaled or aligned" -q > gpurun_out/r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r_tests.log
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2983$n scripts/tp_forward_bench.py 8192 5 sync bf16 > gpurun_out/r_tpfwd_bf16_n$n.json 2> gpurun_out/r_tpfwd_bf16_n$n.err
done
echo done
