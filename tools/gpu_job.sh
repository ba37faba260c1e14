set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
