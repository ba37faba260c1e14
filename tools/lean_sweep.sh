for v in 7 12 0; do
  echo "variant $v"; OEM_LEAN_VARIANT=$v python tools/quick_timing.py --cfg cfg2 --reps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['fit_ms'], d['us_per_iter'])"
done
