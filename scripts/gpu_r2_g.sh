# A/B 2: r01 python + new .so; new tree without NVML; r01 tree again
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
(cd .r01tree && timeout 600 $P --master-port 29760 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-e2e > ../gpurun_out/g_r01.json 2> ../gpurun_out/g_r01.err)
(cd .r01tree_newso && timeout 600 $P --master-port 29761 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu --no-e2e > ../gpurun_out/g_r01_newso.json 2> ../gpurun_out/g_r01_newso.err)
NTP_NO_NVML=1 timeout 600 $P --master-port 29762 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-graph > gpurun_out/g_new_nonvml.json 2> gpurun_out/g_new_nonvml.err
timeout 600 $P --master-port 29763 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-graph > gpurun_out/g_new.json 2> gpurun_out/g_new.err
echo done
