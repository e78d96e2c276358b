"""Summarise an ncu --set full report (read here, no GPU) into a JSON file
under profiles/: the metrics the roofline and DESIGN.md cite.
   python tools/ncu_summary.py REPORT.ncu-rep OUT.json "kernel label" "workload" "capture cmd"
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"]


def main():
    rep, out, kernel, workload, cmd = sys.argv[1:6]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {k: {"value": v[h.index(k)], "unit": u[h.index(k)]} for k in KEYS if k in h}

    def to_bytes(e):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[e["unit"]]
        return float(e["value"].replace(",", "")) * scale
    dram = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
    res = {"kernel": kernel, "workload": workload, "capture": cmd, "round": 2, "metrics": m,
           "dram_bytes_per_launch": dram}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({"dram_bytes_per_launch": dram, "time": m["gpu__time_duration.sum"]}))


if __name__ == "__main__":
    main()
