set -x
mkdir -p gpurun_out
for v in 0 1; do OEM_GRAM_NO_LPT=$v timeout 300 python tools/quick_timing.py --cfg cfg4 --nofit --reps 3 > gpurun_out/qt_cfg4_lpt$v.log 2>&1; done
OEM_GRAM_NO_LPT=1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gram_kernel -c 1 python tools/quick_timing.py --cfg cfg4 --nofit --reps 0 > gpurun_out/ncu_dram_nolpt.log 2>&1
OEM_GRAM_NO_LPT=0 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gram_kernel -c 1 python tools/quick_timing.py --cfg cfg4 --nofit --reps 0 > gpurun_out/ncu_dram_lpt.log 2>&1
