set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_cv.py -m gpu -q > gpurun_out/t_new.log 2>&1; echo tests=$?
OEM_LEAN_VARIANT=6 timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -q -k "cfg1 or cfg2 or sparse or mixed or noncontig or lambda_zero" > gpurun_out/t_v6.log 2>&1; echo tests6=$?
for v in 1 6; do OEM_LEAN_VARIANT=$v timeout 300 python tools/quick_timing.py --cfg cfg2 --reps 2 > gpurun_out/qt_cfg2_v$v.log 2>&1; done
