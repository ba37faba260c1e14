set -x
mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg2 > gpurun_out/bench_cfg2.log 2>&1; echo b=$?
