#!/bin/bash
# One GPU pass (run under gpurun from the repo root): tests, smoke, bench lines, launch lists.
# Usage: tools/gpu_check.sh [tag]   -> gpurun_out/<tag>/...
T=${1:-r2}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --workload lstm --cpu-seconds 5 > $O/bench_lstm.json 2> $O/bench_lstm.err
timeout 300 python bench.py --rank 4 --no-cpu > $O/bench_r4.json 2> $O/bench_r4.err
timeout 300 python bench.py --rank 1 --no-cpu > $O/bench_r1.json 2> $O/bench_r1.err
timeout 400 python bench.py --workload stress --steps 10 --no-cpu > $O/bench_stress.json 2> $O/bench_stress.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_resnet.csv python tools/prof_step.py --steps 4 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_lstm.csv python tools/prof_step.py --workload lstm --rank 4 --steps 4 > /dev/null 2>&1
echo done
