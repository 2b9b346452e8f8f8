# round 2 ncu: launch list of the bench command (N=1) and --set full of the bench kernel (C2, C1)
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
B1="python bench.py --workload mlp-h1024-ffn4096 --steps 3 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/ncu_plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_n1.csv $B > gpurun_out/ncu_launch.log 2>&1
$B > gpurun_out/ncu_plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 3 -c 1 -o gpurun_out/r02_prof_c2 $B > gpurun_out/ncu_full_c2.log 2>&1
$B1 > gpurun_out/ncu_plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 3 -c 1 -o gpurun_out/r02_prof_c1 $B1 > gpurun_out/ncu_full_c1.log 2>&1
echo done
