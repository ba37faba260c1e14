set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -q -k "cfg4 or mixed or sparse" > gpurun_out/t_new.log 2>&1; echo tests=$?
timeout 300 python tools/quick_timing.py --cfg cfg4 --reps 2 > gpurun_out/qt_cfg4.log 2>&1; echo qt=$?
