# Gram pass under different schedules: whole-call time (CUDA events) and the kernel's DRAM
# reads (ncu, one launch). Developer study; results in profiles/cfg4_l2_schedule_r02.md.
# usage: CFG=cfg4 PASS=--plain bash tools/gram_schedule_sweep.sh "ENV=.. ENV2=.." ...
# (CFG=cfg3 PASS= : the fold pass)
mkdir -p gpurun_out
CFG=${CFG:-cfg4}
PASS=${PASS---plain}
run() { echo "== $CFG $1"; env $1 timeout 300 python tools/quick_timing.py --cfg $CFG $PASS --nofit --reps 3 2>&1 | tail -1; env $1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gram_kernel -c 1 --csv python tools/quick_timing.py --cfg $CFG $PASS --nofit --reps 0 2>/dev/null | grep -E 'dram__bytes_read|gpu__time' | awk -F'","' '{print $(NF-2), $NF}'; }
for cfg in "$@"; do run "$cfg"; done
