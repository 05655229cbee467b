#!/bin/bash
# Round-2 profiling pass (run under gpurun from the repo root): bench lines of every
# workload, the reference arm, launch lists with DRAM bytes, and one ncu --set full
# capture of each ResNet-18 / LSTM kernel.  Outputs under gpurun_out/r2prof/.
O=gpurun_out/${PROF_TAG:-r2prof}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1
timeout 400 python bench.py > $O/bench_resnet18_r2.json 2> $O/bench_resnet18_r2.err
timeout 400 python bench.py --rank 1 --no-cpu > $O/bench_resnet18_r1.json 2> $O/bench_resnet18_r1.err
timeout 400 python bench.py --rank 4 --no-cpu > $O/bench_resnet18_r4.json 2> $O/bench_resnet18_r4.err
timeout 400 python bench.py --workload lstm --cpu-seconds 5 > $O/bench_lstm_r4.json 2> $O/bench_lstm_r4.err
timeout 600 python bench.py --workload stress --steps 10 --no-cpu > $O/bench_stress_r8.json 2> $O/bench_stress_r8.err
timeout 400 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_resnet18.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-graph --no-opt > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_lstm.csv python tools/prof_step.py --workload lstm --rank 4 --steps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k1_|k2_|k3_|k4" -c 12 --csv --log-file $O/launches_stress.csv \
    python tools/prof_step.py --workload stress --rank 8 --steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_ef_p|k2_gs|k3_pipe" -s 2 -c 2 \
    -o $O/resnet18_full python tools/prof_step.py --steps 3 > $O/ncu_resnet.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_ef_p|k2_gram|k3_rq|k4_rows" -s 6 -c 6 \
    -o $O/lstm_full python tools/prof_step.py --workload lstm --rank 4 --steps 3 > $O/ncu_lstm.log 2>&1
echo done
