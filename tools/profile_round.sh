#!/bin/bash
# Round profiling on the GPU box (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --workload lstm > gpurun_out/bench_lstm.json 2> gpurun_out/bench_lstm.err
python bench.py --workload stress --steps 10 --no-cpu > gpurun_out/bench_stress.json 2> gpurun_out/bench_stress.err
python bench.py --rank 1 --no-cpu > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
python bench.py --rank 4 --no-cpu > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_ef_p|k2_gs|k3_slab" -s 3 -c 3 \
    -o gpurun_out/prof_full python tools/prof_step.py --steps 3 > gpurun_out/ncu_full.log 2>&1
echo done
