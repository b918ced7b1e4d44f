"""Stall samples and executed instructions per SASS opcode from `ncu --page source --csv` output
(one kernel): python tools/ncu_sass_hist.py source.csv [top_n]"""
import collections
import csv
import sys


def main(path, topn=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot, by, ex, top = 0, collections.Counter(), collections.Counter(), []
    for r in rows:
        if "Warp Stall Sampling (All Samples)" in r:
            hdr = r
            iS, iE, iSrc = r.index("Warp Stall Sampling (All Samples)"), r.index("Instructions Executed"), r.index("Source")
            continue
        if hdr is None or len(r) <= iE:
            continue
        toks = r[iSrc].split()
        if not toks or not r[iS].isdigit():
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        s, e = int(r[iS]), int(r[iE] or 0)
        tot += s
        by[op] += s
        ex[op] += e
        top.append((s, r[iSrc].strip()[:80], e))
    te = sum(ex.values()) or 1
    print(f"total stall samples {tot}, instructions executed {te}")
    for op, s in by.most_common(18):
        print(f"{op:10s} samples {s / max(tot, 1):6.3f}  executed {ex[op] / te:6.3f}")
    top.sort(reverse=True)
    for t in top[:topn]:
        print(t)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
