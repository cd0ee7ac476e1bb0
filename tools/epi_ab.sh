#!/bin/bash
# epilogue decoupling experiments on top of paired MMA iterations (config 2), same box:
for cfg in "" "SPCA_BUILD_NSTG=2" "SPCA_BUILD_PROMO_GP=2" "SPCA_BUILD_KPAIR=0" "SPCA_BUILD_KPAIR=0 SPCA_BUILD_NSTG=2"; do
  env $cfg python -m paper_1704_07669_b200.build --force > /dev/null || { echo "build failed: $cfg"; continue; }
  echo "--- build: ${cfg:-default (KPAIR=1)}"
  bash tools/knobs.sh "X=1" "X=2" "SPCA_TC_UNIT_KB=40"
done
