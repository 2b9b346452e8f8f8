mkdir -p gpurun_out
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/w_bench_n4.json 2> gpurun_out/w_bench_n4.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/w_bench_n2.json 2> gpurun_out/w_bench_n2.err
timeout 300 python scripts/small_variants.py mlp-h1024-ffn4096 100 > gpurun_out/w_small_variants.json 2> gpurun_out/w_small_variants.err
echo done
