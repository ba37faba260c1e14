set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gram.py tests/test_gpu_logistic.py -m gpu -x -q -k "weighted or logistic or logit" > gpurun_out/sc_tests.log 2>&1; echo tests=$?
for r in 1 2; do timeout 200 python tools/quick_timing.py --cfg cfg5 --nofit --reps 5 --noscal > gpurun_out/sc_time_$r.log 2>&1; done
