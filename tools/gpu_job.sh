set -x
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_gram.py -m gpu -x -q -k "weighted" > gpurun_out/pr_tests.log 2>&1; echo tests=$?
Q="timeout 200 python tools/quick_timing.py --cfg cfg5 --nofit --reps 5"
$Q --noscal > gpurun_out/pr_pair.log 2>&1; echo pair=$?
OEM_GRAM_WPAIR=0 $Q --noscal > gpurun_out/pr_nopair.log 2>&1; echo nopair=$?
