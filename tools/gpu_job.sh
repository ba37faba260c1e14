set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_logistic.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
timeout 300 python tools/quick_timing.py --cfg cfg5 --nofit --reps 3 > gpurun_out/qt_cfg5.log 2>&1; echo qt=$?
