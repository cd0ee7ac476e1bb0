#!/bin/bash
# kernel time and DRAM bytes of the pass kernel under chunk / lag knobs (config 2)
#   bash tools/chunk_sweep.sh "SPCA_TC_MIN_ROWS=512 SPCA_TC_CHUNK_MB=20" ...
for kv in "$@"; do
  t=$(env $kv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-pca --no-parity $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms_per_pass'],4), d['roofline']['chunk_rows'])")
  b=$(env $kv ncu --metrics dram__bytes_read.sum --clock-control none -k regex:tc_pass_kernel -s 2 -c 1 python bench.py --steps 3 --warmup 2 --no-e2e --no-pca --no-cpu --no-parity $BENCH_ARGS 2>&1 | grep dram__bytes_read | awk '{print $NF, $(NF-1)}')
  echo "$kv: kernel ms, chunk rows: $t; dram read: $b"
done
