# Scratch job for one-off GPU studies (edit, then run through gpurun):
#   /usr/local/graft/bin/gpurun --timeout 1200 -- 'bash tools/gpu_job.sh'
# Outputs go under gpurun_out/ (merged back, <= 64 MiB). The round's measurement scripts are
# tools/gpu_round.sh (tests, smoke, bench lines, launch lists, reference arm) and
# tools/gpu_ncu_full.sh (one `ncu --set full` capture per Gram workload).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
