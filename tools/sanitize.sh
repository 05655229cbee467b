#!/bin/bash
# compute-sanitizer over every kernel family (run under gpurun): logs in gpurun_out/sanitize/
O=gpurun_out/sanitize; mkdir -p $O; CASES=${SAN_CASES:-resnet18 tall wide}
for c in $CASES; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py $c > $O/${c}_${tool}.log 2>&1
    echo "$c $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${c}_${tool}.log | tail -1)" >> $O/summary.txt
  done
done
cat $O/summary.txt
