set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_stream.py -m gpu -x -q -k "not full_size and not full_n" > gpurun_out/ps_tests.log 2>&1; echo tests=$?
