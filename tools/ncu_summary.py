#!/usr/bin/env python3
"""One-line-per-kernel summary of an ncu report (--page raw --csv): duration, DRAM bytes and
throughput, SM / tensor-pipe activity, achieved occupancy and the top warp-stall reasons.
  python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes_per_launch ...]"""
import csv
import io
import subprocess
import sys

M = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),
    "dram_rd_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_wr_MB": ("dram__bytes_write.sum", 1e-6),
    "dram_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "occ_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
}
UNIT = {"ns": 1, "us": 1e3, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1}


def main():
    rep = sys.argv[1]
    algo = [float(a) for a in sys.argv[2:]]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ix = {k: i for i, k in enumerate(h)}
    stall_cols = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
                  k.endswith("_per_issue_active.ratio") and "not_issued" not in k]
    for n, r in enumerate(rows[2:]):
        out = [r[ix["Kernel Name"]][:70]]
        vals = {}
        for k, (m, sc) in M.items():
            if m not in ix or not r[ix[m]]:
                continue
            v = float(r[ix[m]].replace(",", "")) * UNIT.get(units[ix[m]], 1)
            if k == "dur_us":
                v = v / 1e3
            elif k.endswith("_MB"):
                v = v / 1e6
            vals[k] = v
            out.append(f"{k}={v:.2f}")
        if algo and n < len(algo) and "dur_us" in vals:
            out.append(f"algo_MB={algo[n] / 1e6:.2f} algo_GBs={algo[n] / vals['dur_us'] / 1e3:.0f}")
        st = sorted(((float(r[ix[k]] or 0), k) for k in stall_cols), reverse=True)[:4]
        out.append("stalls/issue=" + ",".join(
            f"{k.split('stalled_')[1].replace('_per_issue_active.ratio', '')}:{v:.2f}" for v, k in st))
        print(" | ".join(out))


if __name__ == "__main__":
    main()
