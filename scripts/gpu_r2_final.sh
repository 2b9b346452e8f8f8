# round 2 final: smoke, whole GPU suite (4 GPUs), bench lines N=1/2/4 (C2) + reference arm
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench_n1.json 2> gpurun_out/f_bench_n1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f_ref_n1.json 2> gpurun_out/f_ref_n1.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/f_bench_n2.json 2> gpurun_out/f_bench_n2.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/f_bench_n4.json 2> gpurun_out/f_bench_n4.err
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/f_pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest_gpu4.log
echo done
