# weighted single-panel pass (cfg5 shape, p as given): job-packing bias against the row warps' sub-partitions
P=$1; shift
for b in "$@"; do echo "p $P bias $b"; OEM_GRAM_RW_BIAS=$b timeout 300 python tools/quick_timing.py --cfg cfg5 --p $P --noscal --reps 3 2>&1 | tail -1; done
