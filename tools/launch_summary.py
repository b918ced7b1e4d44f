"""Per-kernel share of device time from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    for r in rows[hdr_i + 1:]:
        if len(r) <= max(ik, iv, iu):
            continue
        name = r[ik].split("(")[0].replace("void ", "").strip()
        try:
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':48s} {'launches':>8s} {'avg_us':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:48]:48s} {cnt[k]:8d} {tot[k] / cnt[k]:10.1f} {tot[k] / T * 100:6.1f}%")
    print(f"total device time {T / 1e3:.1f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
