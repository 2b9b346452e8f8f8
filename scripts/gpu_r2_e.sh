# round 2, 4 GPUs: whole GPU suite, step overhead vs NCCL uniform, bench N=4 (C2, C1), TP forward N=4, sweep N=4, probes
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29740 scripts/step_overhead.py --rounds 10 > gpurun_out/e_step_overhead.json 2> gpurun_out/e_step_overhead.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/e_bench_c2_n4.json 2> gpurun_out/e_bench_c2_n4.err
timeout 600 python bench.py --gpus 4 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 --no-e2e > gpurun_out/e_bench_c1_n4.json 2> gpurun_out/e_bench_c1_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 scripts/tp_forward_bench.py 8192 5 sync > gpurun_out/e_tpfwd_n4.json 2> gpurun_out/e_tpfwd_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29742 scripts/sweep.py --sync-only > gpurun_out/e_sweep_n4.json 2> gpurun_out/e_sweep_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29743 scripts/small_multi_probe.py > gpurun_out/e_small_probe.json 2> gpurun_out/e_small_probe.err
timeout 900 ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --print-units base --csv --clock-control none python scripts/nvlink_traffic.py gpt-1.3b 1 > gpurun_out/e_nvlink_ncu.csv 2> gpurun_out/e_nvlink_ncu.err
python scripts/nvlink_traffic_summary.py gpurun_out/e_nvlink_ncu.csv 2415919104 > gpurun_out/e_nvlink_summary.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/e_pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest_gpu4.log
echo done
