# round 2: whole GPU suite on 2 GPUs + smoke + sanitizer-free bench sanity
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 1500 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/b_pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest_gpu2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/b_smoke.log
nvidia-smi nvlink -s > gpurun_out/b_nvlink_s.txt 2>&1
nvidia-smi nvlink -gt d > gpurun_out/b_nvlink_gt.txt 2>&1
nvidia-smi nvlink -c > gpurun_out/b_nvlink_c.txt 2>&1
echo done
