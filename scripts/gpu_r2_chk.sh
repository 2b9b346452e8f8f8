mkdir -p gpurun_out
export NCCL_DEBUG=WARN
SECONDS=0; timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --check > gpurun_out/chk_n2.json 2> gpurun_out/chk_n2.err; echo "n2 s=$SECONDS" > gpurun_out/chk_times.txt
SECONDS=0; timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --check --no-e2e > gpurun_out/chk_n4.json 2> gpurun_out/chk_n4.err; echo "n4 s=$SECONDS" >> gpurun_out/chk_times.txt
SECONDS=0; timeout 900 python bench.py --gpus 4 --steps 10 --warmup 3 --check --no-e2e --workload llama3-8b-shaped > gpurun_out/chk_c4_n4.json 2> gpurun_out/chk_c4_n4.err; echo "c4n4 s=$SECONDS" >> gpurun_out/chk_times.txt
timeout 600 python -m pytest tests/test_dist_gpu.py -k "bench_on_shared" -q > gpurun_out/chk_t.log 2>&1; echo "rc=$?" >> gpurun_out/chk_t.log
echo done
