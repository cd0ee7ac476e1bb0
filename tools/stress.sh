#!/bin/bash
# repeated bench runs of one build variant; prints failures' stderr
so=$1; n=${2:-5}
for i in $(seq $n); do
  out=$(SPCA_LIB=$so timeout 300 python bench.py --steps 20 --warmup 3 2>&1); rc=$?
  if [ $rc -ne 0 ]; then echo "run $i rc=$rc"; echo "$out" | tail -8; else echo "run $i ok $(echo "$out" | tail -1 | cut -c1-120)"; fi
done
