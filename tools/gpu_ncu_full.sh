# one `ncu --set full` capture per hot kernel (run only after the same commands exited 0 without ncu)
# usage (through gpurun): bash tools/gpu_ncu_full.sh <tag>; then python tools/ncu_summary.py <tag> name=report ...
set -x
T=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --warmup 0 --steps 1 --e2e-steps 0 --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on -c 1 -f"
for w in cfg4 cfg5 cfg2 cfg3; do timeout 900 $N -k regex:gram_kernel -o gpurun_out/ncu_${T}_gram_$w $B --workload $w > gpurun_out/ncu_${T}_gram_$w.log 2>&1; echo $w=$?; done
timeout 900 $N -k regex:sparse_gram -o gpurun_out/ncu_${T}_sparse $B --workload sparse > gpurun_out/ncu_${T}_sparse.log 2>&1; echo sparse=$?
timeout 900 $N -k regex:fit_active -o gpurun_out/ncu_${T}_active_cfg4 $B --workload cfg4 > gpurun_out/ncu_${T}_active.log 2>&1; echo active=$?
timeout 900 $N -k regex:drule -o gpurun_out/ncu_${T}_drule_cfg4 $B --workload cfg4 > gpurun_out/ncu_${T}_drule.log 2>&1; echo drule=$?
timeout 900 $N -k regex:fit_lean -o gpurun_out/ncu_${T}_lean_cfg2 $B --workload cfg2 > gpurun_out/ncu_${T}_lean.log 2>&1; echo lean=$?
timeout 900 $N -k regex:row_weights -o gpurun_out/ncu_${T}_row_weights python tools/hbm_kernels.py > gpurun_out/ncu_${T}_rw.log 2>&1; echo rw=$?
timeout 900 $N -k regex:logit_grad_kernel -o gpurun_out/ncu_${T}_logit_grad python tools/hbm_kernels.py > gpurun_out/ncu_${T}_lg.log 2>&1; echo lg=$?
