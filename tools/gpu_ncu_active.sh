# ncu --set full of the screened active solver (cfg4, cfg3) on the final code; summarise here with tools/ncu_summary.py
set -x
mkdir -p gpurun_out
B="python bench.py --warmup 0 --steps 1 --e2e-steps 0 --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on -c 1 -f"
for w in cfg4 cfg3; do timeout 600 $N -k regex:fit_active -o gpurun_out/ncu_r02f_active_$w $B --workload $w > gpurun_out/ncu_r02f_active_$w.log 2>&1; echo $w=$?; done
ls -la gpurun_out | tail
python tools/ncu_summary.py r02f active_cfg4_r02f=gpurun_out/ncu_r02f_active_cfg4.ncu-rep active_cfg3_r02f=gpurun_out/ncu_r02f_active_cfg3.ncu-rep > gpurun_out/ncu_summary_r02f.log 2>&1; echo sum=$?
cp profiles/ncu_summary_r02f.json gpurun_out/ 2>/dev/null
for w in cfg4 cfg3; do ncu -i gpurun_out/ncu_r02f_active_$w.ncu-rep --page details --csv > gpurun_out/ncu_r02f_active_${w}_details.csv 2>/dev/null; done
rm -f gpurun_out/*.ncu-rep; du -sh gpurun_out
