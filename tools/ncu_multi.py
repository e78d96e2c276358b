"""Summarise every kernel of an ncu --set full report (read here, no GPU)
into one JSON file under profiles/: time, DRAM bytes and throughput, L2 and
pipe utilisation per launch, plus the achieved HBM bandwidth.
   python tools/ncu_multi.py REPORT.ncu-rep OUT.json "workload" "capture cmd" [hbm_peak_gbs]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "dmma_pipe_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9}


def main():
    rep, out, workload, cmd = sys.argv[1:5]
    peak = float(sys.argv[5]) if len(sys.argv) > 5 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k, m in KEYS.items():
            if m not in h:
                continue
            v, unit = r[h.index(m)].replace(",", ""), u[h.index(m)]
            try:
                x = float(v)
            except ValueError:
                rec[k] = v
                continue
            rec[k] = x * SCALE[unit] if unit in SCALE else x
        t = rec.get("time")
        if t:
            rec["time_ms"] = t * 1e3
            rec["dram_gbs"] = (rec.get("dram_read", 0) + rec.get("dram_write", 0)) / t / 1e9
            if peak:
                rec["dram_frac_of_measured_peak"] = rec["dram_gbs"] / peak
        launches.append(rec)
    json.dump({"workload": workload, "capture": cmd, "hbm_peak_gbs": peak, "launches": launches}, open(out, "w"),
              indent=1)
    for rec in launches:
        print(f"{rec['kernel'][:40]:40s} {rec.get('time_ms', 0):8.3f} ms  {rec.get('dram_gbs', 0):7.0f} GB/s")


if __name__ == "__main__":
    main()
