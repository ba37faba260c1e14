# round measurement: tests, smoke, the bench line of every workload, launch lists, reference arm
# usage (through gpurun): bash tools/gpu_round.sh <round tag, e.g. r02>
set -x
R=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2; lscpu | grep -i 'model name'
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/gpu_tests_$R.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench_${R}_cfg4.log 2>&1; echo bench=$?
for w in cfg2 cfg3 cfg5 sparse; do timeout 600 python bench.py --workload $w --e2e-steps 1 > gpurun_out/bench_${R}_$w.log 2>&1; echo bench_$w=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${R}_cfg4.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_${R}_cfg4.log 2>&1; echo ncu4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_${R}_cfg5.csv python bench.py --workload cfg5 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_${R}_cfg5.log 2>&1; echo ncu5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${R}_sparse.csv python bench.py --workload sparse --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_${R}_sparse.log 2>&1; echo ncus=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${R}_reference.log 2>&1; echo ref=$?
