set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -x -q -k "full_size" --durations=3 > gpurun_out/fs3_tests.log 2>&1; echo tests=$?
