set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 300 python scripts/sync_variants.py 100 > gpurun_out/variants.json 2> gpurun_out/variants.err; echo "rc=$?" >> gpurun_out/variants.err
timeout 300 python scripts/sync_variants.py 20 llama3-8b-shaped > gpurun_out/variants_llama.json 2> gpurun_out/variants_llama.err
echo done
