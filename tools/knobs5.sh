#!/bin/bash
# cfg5 kernel time under tuning-knob environments
for kv in "$@"; do
  v=$(env $kv timeout 200 python bench.py --config cfg5 --steps 3 --warmup 1 --no-e2e --no-pca --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['kernel_ms_per_pass'],2))")
  echo "$kv: ms/step, kernel ms: $v"
done
