set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 300 python tools/quick_timing.py --cfg cfg2 --reps 2 > gpurun_out/qt_cfg2.log 2>&1; echo qt2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fit_cluster -c 1 -o gpurun_out/ncu_path_cfg2 -f python tools/quick_timing.py --cfg cfg2 --reps 0 > gpurun_out/ncu_path_cfg2.log 2>&1; echo ncu=$?
