set -x
mkdir -p gpurun_out
B="python bench.py --warmup 0 --steps 1 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fit_glob_kernel -c 1 -o gpurun_out/ncu_glob_cfg4 -f $B --workload cfg4 > gpurun_out/ncu_glob_cfg4.log 2>&1; echo glob=$?
