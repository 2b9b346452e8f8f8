# 4 GPUs: whole GPU suite on the final kernels, step overhead (prescaled NCCL comparator), C1 bench with the reference-object e2e line
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 600 python bench.py --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 > gpurun_out/n_bench_c1_n1.json 2> gpurun_out/n_bench_c1_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29810 scripts/step_overhead.py --rounds 10 > gpurun_out/n_step_overhead.json 2> gpurun_out/n_step_overhead.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/n_pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/n_pytest_gpu4.log
echo done
