set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_cv.py tests/test_gpu_f3.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
for c in cfg3; do timeout 300 python tools/quick_timing.py --cfg $c --reps 2 > gpurun_out/qt_$c.log 2>&1; echo qt=$?; done
