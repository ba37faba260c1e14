bash tools/gpu_ncu_full.sh r02
python tools/ncu_summary.py r02 gram_cfg4=gpurun_out/ncu_r02_gram_cfg4.ncu-rep gram_cfg5=gpurun_out/ncu_r02_gram_cfg5.ncu-rep gram_cfg2=gpurun_out/ncu_r02_gram_cfg2.ncu-rep gram_cfg3=gpurun_out/ncu_r02_gram_cfg3.ncu-rep sparse=gpurun_out/ncu_r02_sparse.ncu-rep active_cfg4=gpurun_out/ncu_r02_active_cfg4.ncu-rep drule_cfg4=gpurun_out/ncu_r02_drule_cfg4.ncu-rep lean_cfg2=gpurun_out/ncu_r02_lean_cfg2.ncu-rep row_weights_p500=gpurun_out/ncu_r02_row_weights.ncu-rep logit_grad_cfg5=gpurun_out/ncu_r02_logit_grad.ncu-rep > gpurun_out/ncu_summary_r02.log 2>&1
cp profiles/ncu_summary_r02.json gpurun_out/ncu_summary_r02.json
mkdir -p gpurun_out/keep; for f in gram_cfg4 sparse active_cfg4; do cp gpurun_out/ncu_r02_$f.ncu-rep gpurun_out/keep/ 2>/dev/null; done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
