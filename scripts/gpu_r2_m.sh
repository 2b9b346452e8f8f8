# release pattern with one fence: parity (2-GPU dist tests) then latency / sweep / bench
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_signals_gpu.py tests/test_bounds_gpu.py -q > gpurun_out/m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/m_tests.log
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $P --master-port 29800 scripts/probes/signal_latency.py > gpurun_out/m_siglat.json 2> gpurun_out/m_siglat.err
timeout 600 $P --master-port 29801 scripts/small_multi_probe.py > gpurun_out/m_small_probe.json 2> gpurun_out/m_small_probe.err
timeout 900 $P --master-port 29802 scripts/sweep.py --sync-only > gpurun_out/m_sweep_n2.json 2> gpurun_out/m_sweep_n2.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/m_bench_c2_n2.json 2> gpurun_out/m_bench_c2_n2.err
timeout 600 python bench.py --gpus 2 --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 --no-e2e > gpurun_out/m_bench_c1_n2.json 2> gpurun_out/m_bench_c1_n2.err
echo done
