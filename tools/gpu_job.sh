set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_path.py tests/test_gpu_logistic.py tests/test_gpu_cv.py tests/test_gpu_f3.py -m gpu -x -q > gpurun_out/acc_tests.log 2>&1; echo tests=$?
for w in cfg2 cfg3 cfg4 cfg5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/acc_$w.log 2>&1; echo b$w=$?; done
