"""Summarise an ncu report (ncu -i ... --page raw --csv) per kernel: duration, DRAM bytes,
throughput %, occupancy, top stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            try:
                d[h] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
            except ValueError:
                d[h] = v
        recs.append(d)
    return recs


def main(path):
    recs = load(path)
    stall_keys = [k for k in recs[0] if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    for d in recs:
        t = d.get("gpu__time_duration.sum", 0.0)
        rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        st = sorted(((d[k], k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for k in stall_keys if isinstance(d[k], float)), reverse=True)[:4]
        print(f"{d['Kernel Name'][:60]:60s} t={t*1e6:8.1f}us dram R={rd/1e6:8.1f}MB W={wr/1e6:8.1f}MB "
              f"-> {(rd+wr)/t/1e9 if t else 0:7.1f} GB/s dram%={d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f} "
              f"warps%={d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f} regs={d.get('launch__registers_per_thread', 0):.0f} "
              f"fp64%={d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', float('nan')):5.1f} "
              f"stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
