set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_stream.py tests/test_gpu_cv.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
for c in cfg4 cfg3 cfg2 cfg5; do timeout 300 python tools/quick_timing.py --cfg $c --nofit --reps 3 > gpurun_out/qt_$c.log 2>&1; done
