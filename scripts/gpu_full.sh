set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_full.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 600 python bench.py > gpurun_out/bench_full_n1.json 2> gpurun_out/bench_full_n1.err; echo "bench rc=$?" >> gpurun_out/bench_full_n1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
