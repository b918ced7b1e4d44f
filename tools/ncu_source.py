"""Top stalled SASS lines of one kernel in an ncu report (needs -lineinfo for source mapping)."""
import csv
import io
import subprocess
import sys


def main(path, kregex, topn=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{kregex}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # the report may contain several kernels; take the first block
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = []
    for r in rows[hdr_i + 1:]:
        if not r or r[0] == "Kernel Name" or r[0] == "Address":
            break
        data.append(r)
    iS, iSrc, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
    f = lambda v: float(v) if v not in ("", "-") else 0.0
    tot = sum(f(r[iS]) for r in data)
    te = sum(f(r[iE]) for r in data)
    print(f"samples {tot:.0f}  warp-instructions executed {te:.3e}")
    for r in sorted(data, key=lambda r: -f(r[iS]))[:topn]:
        print(f"{f(r[iS]) / tot * 100:5.1f}%  {r[iSrc].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
