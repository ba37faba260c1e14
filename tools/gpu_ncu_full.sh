# one `ncu --set full` capture per hot kernel (run only after the same commands exited 0 without ncu)
set -x
mkdir -p gpurun_out
B="python bench.py --warmup 0 --steps 1 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/ncu_gram_cfg4 -f $B --workload cfg4 > gpurun_out/ncu_full_cfg4.log 2>&1; echo cfg4=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/ncu_gram_cfg5 -f $B --workload cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1; echo cfg5=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/ncu_gram_cfg2 -f $B --workload cfg2 > gpurun_out/ncu_full_cfg2.log 2>&1; echo cfg2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/ncu_gram_cfg3 -f $B --workload cfg3 > gpurun_out/ncu_full_cfg3.log 2>&1; echo cfg3=$?
for w in cfg2 cfg3 cfg5; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$w.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --workload $w > gpurun_out/ncu_launch_$w.log 2>&1; echo launch_$w=$?; done
