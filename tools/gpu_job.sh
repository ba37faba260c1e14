set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_logistic.py tests/test_gpu_stream.py tests/test_gpu_path.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
for c in cfg2 cfg5; do timeout 300 python tools/quick_timing.py --cfg $c --reps 3 > gpurun_out/qt_$c.log 2>&1; echo qt=$?; done
