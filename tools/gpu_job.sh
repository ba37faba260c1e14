set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gram.py -m gpu -q -k "full_size" --durations=5 > gpurun_out/t_new.log 2>&1; echo tests=$?
