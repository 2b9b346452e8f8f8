# round 2: compute-sanitizer memcheck / racecheck / synccheck over smoke(), the
# small sync parity cases, one tcgen05 GEMM shape, a 2-GPU signalled sync, the
# graph steps and the fused row-parallel forward.  Each run bounded by timeout.
mkdir -p gpurun_out/san
export NCCL_DEBUG=WARN PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="compute-sanitizer --error-exitcode 9 --print-limit 50"
run() { name=$1; shift; timeout 1200 "$@" > gpurun_out/san/$name.log 2>&1; echo "rc=$?" >> gpurun_out/san/$name.log; }
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck; do
  run smoke_$tool $CS --tool $tool python -c "$SMOKE"
done
run sync_memcheck $CS --tool memcheck python -m pytest -q tests/test_sync_gpu.py -k "c1_config or edge_cases or weighting or bulk_kernel_variants" -p no:cacheprovider
run sync_racecheck $CS --tool racecheck python -m pytest -q tests/test_sync_gpu.py -k "c1_config or bulk_kernel_variants" -p no:cacheprovider
run sync_synccheck $CS --tool synccheck python -m pytest -q tests/test_sync_gpu.py -k "c1_config or bulk_kernel_variants" -p no:cacheprovider
for w in fwd1 wgrad; do
  for tool in memcheck racecheck synccheck; do
    run gemm_${w}_$tool $CS --tool $tool python scripts/gemm_one.py $w 1
  done
done
run dist2_memcheck $CS --tool memcheck --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 scripts/dist_check.py 4 3 f32 2 three
run dist2_graph_memcheck $CS --tool memcheck --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 scripts/dist_check.py 4 3 f32 3 graph
run dist2_synccheck $CS --tool synccheck --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29733 scripts/dist_check.py 4 3 bf16 2 fused
run tpfwd2_memcheck $CS --tool memcheck --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29734 scripts/tp_forward_check.py push sync 512
for f in gpurun_out/san/*.log; do echo "== $f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|rc=' $f | tr '\n' ' ')"; done > gpurun_out/san/summary.txt
echo done
