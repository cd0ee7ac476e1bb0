#!/bin/bash
# kernel time under tuning-knob environments: tools/knobs.sh "SPCA_TC_LAG=3" "SPCA_TC_CHUNK_MB=20" ...
# (BENCH_ARGS adds bench.py flags, e.g. "--config cfg3"); each run bounded by 90 s
for kv in "$@"; do
  v=$(env $kv timeout 90 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-pca --no-parity $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys
try:
    d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_pass'],4))
except Exception:
    print('failed / timed out')")
  echo "$kv: ms/step, kernel ms: $v"
done
