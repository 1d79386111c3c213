#!/bin/bash
# Round profile set (run on the GPU box from the repo root):
#   launch list of a bench step, ncu --set full of the timed step's key-select / direct-scan /
#   group-tables / refine kernels (summarised; the scan's DRAM traffic goes
#   to profiles/ncu_scan_traffic.json for bench.py's roofline.traffic).
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-comparator"
$B > "$OUT/plain.log" 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 200 --csv \
    --log-file "$OUT/launches.csv" $B > "$OUT/ncu_launches.log" 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_key_select|k_scan_direct|k_group_tables|k_refine_topk|k_threshold" -s 10 -c 5 \
    -o "$OUT/prof_full" $B > "$OUT/ncu_full.log" 2>&1
python scripts/ncu_summary.py "$OUT/prof_full.ncu-rep" "$B" > "$OUT/ncu_full_metrics.json"
python - "$OUT/ncu_full_metrics.json" "$OUT/ncu_scan_traffic.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
k = [x for x in d["kernels"] if "k_scan_direct" in x["kernel"]][0]
json.dump({"config": "c2", "kernel": k["kernel"], "traffic_bytes": k["traffic_bytes"],
           "duration_us": k["duration_us"], "capture": d["capture"]}, open(sys.argv[2], "w"), indent=1)
PY
echo done
