#!/bin/bash
# kernel time of one config under tuning-knob environments: tools/knobsc.sh cfg3 "K=V" ...
cfg=$1; shift
for kv in "$@"; do
  v=$(env $kv timeout 300 python bench.py --config $cfg --steps 5 --warmup 2 --no-e2e --no-pca --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_pass'],3), round(d['roofline']['frac'],3))")
  echo "$cfg $kv: ms/step, kernel ms, frac: $v"
done
