set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --no-cpu --e2e-steps 6 > gpurun_out/bench_e2e_layer.json 2> gpurun_out/bench_e2e_layer.err
NTP_E2E_SEGS_PER_PIECE=1 timeout 600 python bench.py --steps 50 --no-cpu --e2e-steps 6 > gpurun_out/bench_e2e_seg.json 2> gpurun_out/bench_e2e_seg.err
echo done
