#!/bin/bash
# A/B kernel time of two builds, alternating: tools/ab.sh a.so b.so [rounds] (BENCH_ARGS: extra bench flags)
a=$1; b=$2; n=${3:-2}
for i in $(seq $n); do
  for so in $a $b; do
    v=$(SPCA_LIB=$so python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-pca $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_pass'],4))")
    echo "$so: ms/step, kernel ms: $v"
  done
done
