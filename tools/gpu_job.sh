set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py -m gpu -x -q -k "full_n_column_subset_cfg4 or weighted_full_size_cfg5" --durations=3 > gpurun_out/fs2_tests.log 2>&1; echo tests=$?
