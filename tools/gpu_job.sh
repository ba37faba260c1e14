set -x
mkdir -p gpurun_out
for v in 5 10; do OEM_LEAN_VARIANT=$v timeout 600 python bench.py --workload cfg3 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/ly3_$v.log 2>&1; echo c3v$v=$?; done
OEM_LEAN_VARIANT=10 timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_cv.py -m gpu -x -q -k "cfg3 or boundaries or cv" > gpurun_out/ly_tests10.log 2>&1; echo t10=$?
