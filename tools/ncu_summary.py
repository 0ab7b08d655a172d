"""Summarise an ncu report (`--set full`) into a compact JSON per kernel launch:
duration, DRAM bytes, pipe utilisation, issue activity, occupancy and the top
stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fma_pipe_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fmaheavy_pipe_active_pct": ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "grid_size": ("launch__grid_size", 1.0),
    "block_size": ("launch__block_size", 1.0),
    "waves_per_sm": ("launch__waves_per_multiprocessor", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "smem_bank_conflicts_ld": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1.0),
    "smem_bank_conflicts_st": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", 1.0),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1.0),
}


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")]}
        for k, (metric, scale) in KEYS.items():
            if metric in hdr:
                v = _num(d[hdr.index(metric)])
                u = units[hdr.index(metric)]
                if v is not None and metric == "gpu__time_duration.sum":
                    v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, scale)
                elif v is not None and metric.startswith("dram__bytes"):
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
                elif v is not None and metric == "sm__cycles_elapsed.avg.per_second":
                    v = v * {"Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}.get(u, 1.0)
                rec[k] = v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                v = _num(d[i])
                if v and v > 0.05:
                    stalls.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], round(v, 3)))
        stalls.sort(key=lambda x: -x[1])
        rec["top_stalls_per_issue"] = stalls[:8]
        if rec.get("dram_read_bytes") is not None:
            rec["dram_bytes_per_launch"] = rec["dram_read_bytes"] + (rec.get("dram_write_bytes") or 0)
        res.append(rec)
    return res


if __name__ == "__main__":
    r = summarise(sys.argv[1])
    s = json.dumps(r, indent=1)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(s + "\n")
    print(s)
