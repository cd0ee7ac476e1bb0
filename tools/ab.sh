#!/bin/bash
# A/B timing of build variants: tools/ab.sh variants/*.so  (bench cfg2, 2 rounds interleaved)
for r in 1 2; do
  for so in "$@"; do
    v=$(SPCA_LIB=$so python bench.py --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_pass'],4))")
    echo "$so: ms/step, kernel ms: $v"
  done
done
