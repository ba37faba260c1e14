set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -m gpu -x -q > gpurun_out/st_tests.log 2>&1; echo tests=$?
