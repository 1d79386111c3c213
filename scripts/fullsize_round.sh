#!/bin/bash
# Full-size parity + phase runs of BASELINE configs 2-5 (GPU box, repo root).
set -u
OUT=${1:-gpurun_out/fs}
mkdir -p "$OUT"
for c in c2 c3 c4 c5; do
  timeout 1500 python scripts/fullsize.py --config $c --check 64 > "$OUT/$c.json" 2> "$OUT/$c.err"
  echo "$c rc=$?"
done
DPQ_TC_TABLES=0 timeout 1200 python scripts/fullsize.py --config c5 --check 8 > "$OUT/c5_lazy.json" 2> "$OUT/c5_lazy.err"
echo "c5_lazy rc=$?"
