"""Predicted load balance of bench.py's fixed 48-problem config-3 batch at 2/4/8 ranks from a
1-GPU bench line's measured per-problem device times (config.problem_ms_step1): each rank's time
= the sum over its shard (dist.config3_shard, the assignment bench.py uses), efficiency =
total / (N * max rank time).  A prediction for the driver's scaling run (which measures it); it
ignores clock droop with 8 busy GPUs.  python tools/shard_balance.py bench_line.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import dist as D  # noqa: E402


def main(path):
    line = json.loads(open(path).read().strip().splitlines()[-1])
    cfg = line["config"]
    t = dict(zip(cfg["problems"], cfg["problem_ms_step1"]))
    tot = sum(t.values())
    print(f"48 problems, {tot:.1f} ms of device time in step 1 (1 GPU)")
    for n in (2, 4, 8):
        ranks = [sum(t[f"m{m}R{R:g}"] for m, R in D.config3_shard(n, r)) for r in range(n)]
        print(f"N={n}: rank ms {[round(x, 1) for x in ranks]}  max/mean {max(ranks) / (tot / n):.4f}  "
              f"predicted efficiency {tot / (n * max(ranks)):.4f}")


if __name__ == "__main__":
    main(sys.argv[1])
