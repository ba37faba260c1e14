set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_logistic.py tests/test_gpu_stream.py tests/test_gpu_poison.py -m gpu -x -q > gpurun_out/wf_tests.log 2>&1; echo tests=$?
for w in cfg2 cfg5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --e2e-steps 1 --steps 3 > gpurun_out/wf_$w.log 2>&1; echo b$w=$?; done
