set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
for c in cfg4 cfg3; do timeout 300 python tools/quick_timing.py --cfg $c --reps 3 --nofit > gpurun_out/qt_$c.log 2>&1; echo qt=$?; done
