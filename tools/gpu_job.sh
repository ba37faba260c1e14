set -x
mkdir -p gpurun_out
for v in 3 4; do OEM_GLOB_VARIANT=$v timeout 600 python bench.py --workload cfg4 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/g4_$v.log 2>&1; echo v$v=$?; done
OEM_GLOB_VARIANT=4 timeout 600 python -m pytest tests/test_gpu_path.py -m gpu -x -q -k "cfg4 or boundaries or mixed or sparse_group" > gpurun_out/g4_tests.log 2>&1; echo t=$?
