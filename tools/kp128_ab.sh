#!/bin/bash
# paired MMA-warp iterations for l_pad 128 as well (SPCA_KPAIR=2), same box
for cfg in "SPCA_BUILD_KPAIR=2" "SPCA_BUILD_KPAIR=1"; do
  env $cfg python -m paper_1704_07669_b200.build --force > /dev/null || { echo "build failed: $cfg"; continue; }
  echo "--- build: $cfg"
  BENCH_ARGS="--config cfg3" bash tools/knobs.sh "X=1" "X=2"
  BENCH_ARGS="--config cfg5" bash tools/knobs.sh "X=1"
  if [ "$cfg" = "SPCA_BUILD_KPAIR=2" ]; then timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_alg.py -x -q 2>&1 | tail -2; fi
done
