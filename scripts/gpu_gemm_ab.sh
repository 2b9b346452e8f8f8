# A/B of GEMM builds/variants at base clocks (ncu --clock-control base): kernel
# efficiency without the power cap.  usage: bash scripts/gpu_gemm_ab.sh "<label>=<env> ..."
mkdir -p gpurun_out/ab
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for v in "$@"; do
  label=${v%%=*}; envs=${v#*=}
  for n in 4779 3584; do
    env $envs timeout 300 ncu --clock-control base --metrics $M -k "regex:gemm_kernel|nvjet|cutlass" --csv \
      python scripts/gemm_pair.py all 3 $n > gpurun_out/ab/${label}_$n.csv 2> gpurun_out/ab/${label}_$n.err
    echo "$label $n rc=$?"
  done
done
