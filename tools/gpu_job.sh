set -x
mkdir -p gpurun_out
OEM_POISON=1 timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/poison.log 2>&1; echo poison=$?; tail -3 gpurun_out/poison.log
