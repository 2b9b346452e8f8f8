# repeatability: the default bench line at N=1/2/4, five runs each, interleaved (device numbers only)
mkdir -p gpurun_out/rep
export NCCL_DEBUG=WARN
for i in 1 2 3 4 5; do
for n in 1 2 4; do
timeout 300 python bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/rep/n${n}_$i.json 2> gpurun_out/rep/n${n}_$i.err
done
done
echo done
