# End-of-session check on 4 GPUs: the whole GPU suite, N=2 / N=4 bench lines and
# the reference arm under torchrun.
set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2969$n bench.py --gpus $n --steps 20 --warmup 3 --e2e-steps 8 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench n=$n rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29681 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > gpurun_out/bench_ref_n4.json 2> gpurun_out/bench_ref_n4.err
echo "ref rc=$?"
