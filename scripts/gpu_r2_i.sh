# 4 GPUs: TP forward (reduce-broadcast) tests + bench at N=2/N=4, bench N=4 lines without NVML, small probe
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_dist_gpu.py -k "row_parallel" -q > gpurun_out/i_pytest_tp.log 2>&1; echo "rc=$?" >> gpurun_out/i_pytest_tp.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29780 scripts/tp_forward_bench.py 8192 5 sync > gpurun_out/i_tpfwd_n4.json 2> gpurun_out/i_tpfwd_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 scripts/tp_forward_bench.py 8192 5 sync > gpurun_out/i_tpfwd_n2.json 2> gpurun_out/i_tpfwd_n2.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/i_bench_c2_n4.json 2> gpurun_out/i_bench_c2_n4.err
timeout 600 python bench.py --gpus 4 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 > gpurun_out/i_bench_c1_n4.json 2> gpurun_out/i_bench_c1_n4.err
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --workload llama3-8b-shaped --no-e2e > gpurun_out/i_bench_c4_n4.json 2> gpurun_out/i_bench_c4_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29782 scripts/small_multi_probe.py > gpurun_out/i_small_probe.json 2> gpurun_out/i_small_probe.err
echo done
