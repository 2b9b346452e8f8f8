set -x
mkdir -p gpurun_out
for v in 1 3 2; do
  NTP_SYNC_KERNEL=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2942$v bench.py --gpus 2 --steps 100 > gpurun_out/bench_n2_v$v.json 2> gpurun_out/bench_n2_v$v.err
done
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_linear_gpu.py -q -x -k "epilogues or tensor_core" > gpurun_out/memcheck_linear.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_linear.log
echo done
