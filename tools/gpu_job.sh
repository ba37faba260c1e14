set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg4 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/gv_2.log 2>&1; echo v2=$?
OEM_GLOB_VARIANT=3 timeout 600 python bench.py --workload cfg4 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/gv_3.log 2>&1; echo v3=$?
OEM_GLOB_VARIANT=3 timeout 900 python -m pytest tests/test_gpu_path.py -m gpu -x -q -k "cfg4 or boundaries or mixed or sparse_group or batched" > gpurun_out/gv_tests3.log 2>&1; echo t3=$?
