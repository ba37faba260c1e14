# one `ncu --set full` capture per hot kernel (run only after the same commands exited 0 without ncu)
set -x
mkdir -p gpurun_out
B="python bench.py --warmup 0 --steps 1 --e2e-steps 0 --no-cpu-baseline"
for w in cfg4 cfg5 cfg2 cfg3; do timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 1 -o gpurun_out/ncu_gram_$w -f $B --workload $w > gpurun_out/ncu_full_$w.log 2>&1; echo $w=$?; done
