#!/bin/bash
# converter groups A/B on the GPU box: default build (3 groups for l_pad 64), then a 2-group rebuild
bash tools/knobs.sh "X=1" "SPCA_TC_DEBUG=18446" "SPCA_TC_DEBUG=18432" "SPCA_TC_DEBUG=16384" "X=2"
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
SPCA_BUILD_GROUPS=2 python -m paper_1704_07669_b200.build --force > /dev/null
echo "--- 2 groups"
bash tools/knobs.sh "X=1" "SPCA_TC_DEBUG=18446" "X=2"
