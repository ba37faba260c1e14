set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -x -q -k "full_size" --durations=5 > gpurun_out/fs_tests.log 2>&1; echo tests=$?
