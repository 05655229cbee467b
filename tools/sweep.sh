#!/bin/bash
# Environment sweep of plan knobs (run under gpurun): tools/sweep.sh <tag> "<bench args>" "ENV=a ENV2=b" "ENV=c" ...
T=$1; shift; ARGS=$1; shift
O=gpurun_out/$T; mkdir -p $O
for cfg in "$@"; do
  name=$(echo "$cfg" | tr ' =/' '_-_')
  env $cfg timeout 300 python bench.py --no-cpu $ARGS > $O/$name.json 2> $O/$name.err
  python - "$O/$name.json" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:40s} step {d['value']*1e3:8.2f} us  b2b {d['config']['back_to_back_ms']*1e3:8.2f}  frac {d['step_roofline']['frac']:.4f}  k {d['kernels_ms']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
