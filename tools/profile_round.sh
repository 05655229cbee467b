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
ncu --set full --clock-control none --import-source on -k regex:"k1_ef_p|k2_gs|k3_slab|k3_pipe" -s 3 -c 3 \
    -o gpurun_out/prof_full python tools/prof_step.py --steps 3 > gpurun_out/ncu_full.log 2>&1

ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k1_|k2_|k3_|k4" -s 9 -c 9 --csv --log-file gpurun_out/launches_stress.csv \
    python tools/prof_step.py --workload stress --rank 8 --steps 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k1_|k2_|k3_|k4" -s 12 -c 12 --csv --log-file gpurun_out/launches_lstm.csv \
    python tools/prof_step.py --workload lstm --rank 4 --steps 4 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo done2
