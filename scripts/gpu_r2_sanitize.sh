# round 2: ONE compute-sanitizer tool per gpurun call (B200_PROFILING.md):
#   bash scripts/gpu_r2_sanitize.sh memcheck|racecheck|synccheck
# over smoke(), the small sync parity cases, two tcgen05 GEMM shapes and (memcheck,
# synccheck) a 2-GPU signalled sync, CUDA-graph steps and the fused TP forward.
tool=${1:-memcheck}
mkdir -p gpurun_out/san
export NCCL_DEBUG=WARN PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50"
run() { name=$1; shift; timeout 1500 "$@" > gpurun_out/san/${name}_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san/${name}_$tool.log; }
run smoke $CS python -c 'import __graft_entry__ as g; g.smoke()'
run sync $CS python -m pytest -q tests/test_sync_gpu.py -k "c1_config or bulk_kernel_variants or edge_cases" -p no:cacheprovider
run gemm_fwd1 $CS python scripts/gemm_one.py fwd1 1
run gemm_wgrad $CS python scripts/gemm_one.py wgrad 1
if [ "$tool" != racecheck ]; then
  run dist2 $CS --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 scripts/dist_check.py 4 3 f32 2 three
  run dist2_graph $CS --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 scripts/dist_check.py 4 3 bf16 3 graph_fused
  run tpfwd2 $CS --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29734 scripts/tp_forward_check.py push sync 512
fi
for f in gpurun_out/san/*_$tool.log; do echo "== $f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Hazard|rc=' $f | sort | uniq -c | tr '\n' ' ')"; done > gpurun_out/san/summary_$tool.txt
echo done
