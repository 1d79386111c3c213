#!/bin/bash
# Round profile set (run on the GPU box from the repo root):
#   bench line, reference-arm line, ncu launch list, ncu --set full of the
#   timed step's scan / group-tables / refine kernels, ncu --set full of the
#   tensor-core encoder, host-API (e2e) segment trace.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
python bench.py --impl reference > "$OUT/ref.json" 2> "$OUT/ref.err"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > "$OUT/plain.log" 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 200 --csv \
    --log-file "$OUT/launches.csv" $B > "$OUT/ncu_launches.log" 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_scan_emit|k_group_tables|k_refine_topk" -s 3 -c 3 \
    -o "$OUT/prof_full" $B > "$OUT/ncu_full.log" 2>&1
E="python scripts/encode_bench.py --n 1000000 --n-torch 10000 --reps 1"
$E > "$OUT/enc_plain.log" 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_encode_tc -s 1 -c 1 \
    -o "$OUT/enc_full" $E > "$OUT/enc_ncu.log" 2>&1
DPQ_HOST_TRACE=1 python scripts/diag_e2e.py > "$OUT/e2e_diag.log" 2>&1
echo done
