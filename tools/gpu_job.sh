set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fit_glob -c 1 -o gpurun_out/ncu_glob_cfg4b -f python tools/quick_timing.py --cfg cfg4 --reps 0 > gpurun_out/ncu_glob.log 2>&1; echo ncu=$?
