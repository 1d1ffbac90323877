"""Summarise an ncu --set full report (raw page) per kernel launch."""
import csv
import subprocess
import sys


def f(v):
    try:
        return float(v)
    except Exception:
        return 0.0


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1])) if len(rows) > 1 else {}
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), f(v))
                     for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled")
                     and k.endswith("per_issue_active.ratio")), key=lambda kv: -kv[1])
        out.append({
            "kernel": d.get("Kernel Name", "")[:70],
            "time": f(d.get("gpu__time_duration.sum")),
            "dmma_pipe_pct": f(d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")),
            "dram_read": f(d.get("dram__bytes_read.sum")),
            "dram_write": f(d.get("dram__bytes_write.sum")),
            "dram_unit": units.get("dram__bytes_read.sum"),
            "time_unit": units.get("gpu__time_duration.sum"),
            "dram_pct": f(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
            "issue_pct": f(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active")),
            "regs": d.get("launch__registers_per_thread"),
            "smem_conflicts_ld": f(d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")),
            "smem_conflicts_st": f(d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum")),
            "stalls_per_issue": [(k, round(v, 2)) for k, v in st[:6]],
        })
    return out


if __name__ == "__main__":
    import json
    for rep in sys.argv[1:]:
        print(rep)
        for k in summarise(rep):
            print(json.dumps(k))
