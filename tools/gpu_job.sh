set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -q -k "variant_boundaries" > gpurun_out/t_new.log 2>&1; echo tests=$?
