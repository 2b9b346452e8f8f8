# A/B: bench N=2 (C2) with the r01 tree vs this tree (graph / no-graph), same box; C1 N=2 variants
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
(cd .r01tree && timeout 600 $P --master-port 29750 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-e2e > ../gpurun_out/f_r01_n2.json 2> ../gpurun_out/f_r01_n2.err)
timeout 600 $P --master-port 29751 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-graph > gpurun_out/f_nograph_n2.json 2> gpurun_out/f_nograph_n2.err
timeout 600 $P --master-port 29752 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e > gpurun_out/f_graph_n2.json 2> gpurun_out/f_graph_n2.err
(cd .r01tree && timeout 600 $P --master-port 29753 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-e2e > ../gpurun_out/f_r01_n2b.json 2> ../gpurun_out/f_r01_n2b.err)
timeout 600 $P --master-port 29754 scripts/small_multi_probe.py > gpurun_out/f_small_probe.json 2> gpurun_out/f_small_probe.err
echo done
