"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel class
from one `ncu --set full` capture -> profiles/traffic_rNN.json (read by bench.py's roofline).
Usage: python tools/traffic.py report.ncu-rep profiles/traffic_r01.json"""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

CLASSES = [("kp_thermal3d", "K"), ("kp_elastic3d", "K"), ("xfwd_kernel", "xfwd"), ("xfwd256", "xfwd"),
           ("xfwd512", "xfwd"), ("ypass_kernel", "ypass"), ("ypass256", "ypass"), ("ypass512", "ypass"),
           ("gpass_z_kernel", "gpass"), ("gpass256", "gpass"), ("gpass512", "gpass"), ("gpass_y2d", "gpass"),
           ("xinv_kernel", "xinv"), ("xinv512", "xinv"), ("scalar_kernel", "scalar"), ("dstz_kernel", "dstz")]


def main(rep, out):
    acc = defaultdict(list)
    for d in load(rep):
        name = d["Kernel Name"]
        cls = next((c for p, c in CLASSES if p in name), None)
        if cls is None:
            continue
        acc[cls].append(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0))
    res = {k: round(sum(v) / len(v)) for k, v in acc.items()}
    res["_source"] = f"ncu --set full capture {os.path.basename(rep)} (tools/profile_solve.py, 256^3 thermal, 3 loads); mean over captured launches"
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
