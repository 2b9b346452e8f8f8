# round 2: graph-step fixes, TP forward (2 GPUs), N=2 bench lines, sweep, NVLink traffic (ncu), small variants
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_dist_gpu.py -k "graph or row_parallel or aligned" tests/test_dropin_gpu.py -q > gpurun_out/d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d_pytest.log
timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 --no-e2e > gpurun_out/d_bench_c1_n2.json 2> gpurun_out/d_bench_c1_n2.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/d_bench_c2_n2.json 2> gpurun_out/d_bench_c2_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29720 scripts/sweep.py --sync-only > gpurun_out/d_sweep_n2.json 2> gpurun_out/d_sweep_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29721 scripts/tp_forward_bench.py 8192 5 sync > gpurun_out/d_tpfwd_n2.json 2> gpurun_out/d_tpfwd_n2.err
timeout 300 python scripts/small_variants.py mlp-h1024-ffn4096 100 > gpurun_out/d_small_variants.json 2> gpurun_out/d_small_variants.err
timeout 900 ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --print-units base --csv --clock-control none python scripts/nvlink_traffic.py gpt-1.3b 1 > gpurun_out/d_nvlink_ncu.csv 2> gpurun_out/d_nvlink_ncu.err
python scripts/nvlink_traffic_summary.py gpurun_out/d_nvlink_ncu.csv 2415919104 > gpurun_out/d_nvlink_summary.json 2>&1
echo done
