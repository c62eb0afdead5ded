"""Summarise an ncu report (raw page) into a small JSON/markdown table for profiles/."""
import csv
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1),
    "fp64_pipe_pct_active": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "dfma_thread_inst_per_cycle": ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed", 1),
    "dmul_thread_inst_per_cycle": ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed", 1),
    "dadd_thread_inst_per_cycle": ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", 1),
    "dram_read_MB": ("dram__bytes_read.sum", 1),
    "dram_write_MB": ("dram__bytes_write.sum", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "sm_clock_GHz": ("smsp__cycles_elapsed.avg.per_second", 1),
}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[h.index("Kernel Name")]}
        for k, (m, scale) in KEYS.items():
            if m in h:
                try:
                    v = float(row[h.index(m)])
                    u = units[h.index(m)]
                    if m.startswith("dram__bytes"):
                        v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                    if m == "gpu__time_duration.sum":
                        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "us": 1.0}.get(u, 1.0)
                    d[k] = v
                except ValueError:
                    pass
        stalls = {}
        for i, m in enumerate(h):
            if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
                try:
                    stalls[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(row[i])
                except ValueError:
                    pass
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
