set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_cv.py tests/test_gpu_f3.py tests/test_gpu_logistic.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
timeout 300 python tools/quick_timing.py --cfg cfg2 --reps 2 > gpurun_out/qt_cfg2.log 2>&1
