set -x
mkdir -p gpurun_out
for rep in 1 2; do
for v in new head; do
  if [ $v = head ]; then cp paper_1801_09661_b200/liboem.so /tmp/liboem_new.so; cp liboem_head.so paper_1801_09661_b200/liboem.so; fi
  for w in cfg2 cfg3 cfg4; do timeout 600 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/v_${v}_${w}_$rep.log 2>&1; echo $v$w=$?; done
  if [ $v = head ]; then cp /tmp/liboem_new.so paper_1801_09661_b200/liboem.so; fi
done
done
