set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_logistic.py -m gpu -x -q > gpurun_out/w_tests.log 2>&1; echo tests=$?
Q="timeout 300 python tools/quick_timing.py --cfg cfg5 --nofit --reps 3"
$Q > gpurun_out/y_scal.log 2>&1; echo scal=$?
$Q --noscal > gpurun_out/y_noscal.log 2>&1; echo noscal=$?
timeout 600 python bench.py --workload cfg5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5.log 2>&1; echo bench5=$?
