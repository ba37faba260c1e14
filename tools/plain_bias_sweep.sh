for b in 0 1 2 3 4 6; do echo "bias $b"; OEM_GRAM_RW_BIAS=$b timeout 300 python tools/quick_timing.py --cfg cfg2 --nofit --reps 5 2>&1 | tail -1; done
for b in 0 2 4 8; do echo "p200 plain bias $b"; OEM_GRAM_RW_BIAS=$b timeout 300 python tools/quick_timing.py --cfg cfg5 --plain --nofit --reps 3 2>&1 | tail -1; done
