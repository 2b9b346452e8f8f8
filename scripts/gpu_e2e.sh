set -x
mkdir -p gpurun_out
for l in 1 2 4; do
NTP_E2E_LAYERS_PER_PIECE=$l timeout 600 python bench.py --steps 50 --no-cpu --e2e-steps 6 > gpurun_out/bench_e2e_$l.json 2> gpurun_out/bench_e2e_$l.err
done
echo done
