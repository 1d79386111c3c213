"""Summarise an `ncu --set full` report into the JSON kept under profiles/.

    python scripts/ncu_summary.py REPORT.ncu-rep "capture command" > profiles/NAME.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "tensor_pipe_active_pct_elapsed": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "sm_cycles": ("sm__cycles_elapsed.avg", 1),
    "sm_mhz": ("sm__cycles_elapsed.avg.per_second", 1e-6),
    "tmem_load_insts": ("smsp__sass_inst_executed_op_tmem_ldt.sum", 1),
}


def main():
    rep, cap = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, data = rows[0], rows[2:]
    out = []
    for r in data:
        k = {"kernel": r[head.index("Kernel Name")]}
        for key, (name, scale) in METRICS.items():
            if name in head:
                v = r[head.index(name)].replace(",", "")
                try:
                    k[key] = round(float(v) * scale, 6)
                except ValueError:
                    pass
        if "dram_read_MB" in k and "dram_write_MB" in k:
            k["traffic_bytes"] = int(round((k["dram_read_MB"] + k["dram_write_MB"]) * 1e6))
        out.append(k)
    print(json.dumps({"capture": cap, "kernels": out}, indent=1))


if __name__ == "__main__":
    main()
