set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_logistic.py -m gpu -x -q -k "weighted or logistic or logit" > gpurun_out/z_tests.log 2>&1; echo tests=$?
Q="timeout 300 python tools/quick_timing.py --cfg cfg5 --nofit --reps 5"
for v in new base; do
  if [ $v = base ]; then cp paper_1801_09661_b200/liboem.so /tmp/liboem_new.so; cp liboem_base.so paper_1801_09661_b200/liboem.so; fi
  $Q > gpurun_out/z_${v}_scal.log 2>&1
  $Q --noscal > gpurun_out/z_${v}_noscal.log 2>&1
  timeout 600 python bench.py --workload cfg5 --no-cpu-baseline --e2e-steps 0 --steps 2 > gpurun_out/z_${v}_bench.log 2>&1; echo b$v=$?
  if [ $v = base ]; then cp /tmp/liboem_new.so paper_1801_09661_b200/liboem.so; fi
done
