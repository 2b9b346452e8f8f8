mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 --workload mlp-h1024-ffn4096 > gpurun_out/p_bench_c1_n1.json 2> gpurun_out/p_bench_c1_n1.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/p_bench_c2_n1.json 2> gpurun_out/p_bench_c2_n1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/p_ref_c2.json 2> gpurun_out/p_ref_c2.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/p_smoke.log
echo done
