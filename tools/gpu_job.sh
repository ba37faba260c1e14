set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
for c in cfg1 cfg2; do timeout 300 python tools/quick_timing.py --cfg $c --reps 2 > gpurun_out/qt_$c.log 2>&1; echo qt=$?; done
