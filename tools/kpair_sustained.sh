#!/bin/bash
# tie-breaker for SPCA_KPAIR at config 2: sustained (power-capped) rate over 300 back-to-back passes, same box
for cfg in "SPCA_BUILD_KPAIR=1" "SPCA_BUILD_KPAIR=0" "SPCA_BUILD_KPAIR=1" "SPCA_BUILD_KPAIR=0"; do
  env $cfg python -m paper_1704_07669_b200.build --force > /dev/null || { echo "build failed: $cfg"; continue; }
  for k in 20 300; do
    python bench.py --steps $k --warmup 5 --no-e2e --no-cpu --no-pca --no-parity 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$cfg steps', d['steps'], 'ms/step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms_per_pass'],4), 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'W', d['clocks'].get('power_w_max'))"
  done
done
