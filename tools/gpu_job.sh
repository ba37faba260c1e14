set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_f3.py tests/test_gpu_cv.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
timeout 300 python tools/quick_timing.py --cfg cfg4 --reps 2 > gpurun_out/qt_cfg4.log 2>&1
OEM_PATH_SOLVER=batched timeout 300 python tools/quick_timing.py --cfg cfg4 --reps 2 > gpurun_out/qt_cfg4_b.log 2>&1
