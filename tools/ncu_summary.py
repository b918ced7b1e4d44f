"""One-line ncu summaries (time, DRAM bytes, occupancy, issue, FP64 pipe, smem wavefronts, top stalls)
per kernel of .ncu-rep files: python tools/ncu_summary.py a.ncu-rep [...]"""
import csv
import subprocess
import sys

KEYS = [('gpu__time_duration.sum', 't_us'), ('dram__bytes_read.sum', 'dramR_MB'), ('dram__bytes_write.sum', 'dramW_MB'),
        ('sm__warps_active.avg.pct_of_peak_sustained_active', 'warps%'),
        ('smsp__issue_active.avg.pct_of_peak_sustained_active', 'issue%'),
        ('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'fp64%'),
        ('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed', 'smem_wf%'),
        ('launch__registers_per_thread', 'regs')]
_BYTES = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'B': 1.0, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}
_TIME = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3, 'second': 1e6, 's': 1e6}


def _rows(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def load(rep):
    """Per launch: dict with the kernel name and the DRAM byte counts (bytes) and time (us) as floats."""
    h, u, body = _rows(rep)
    res = []
    for v in body:
        d = dict(zip(h, v))
        un = dict(zip(h, u))
        r = {'Kernel Name': d['Kernel Name']}
        for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
            r[k] = float(d[k].replace(',', '')) * _BYTES.get(un[k], 1.0)
        r['t_us'] = float(d['gpu__time_duration.sum'].replace(',', '')) * _TIME.get(un['gpu__time_duration.sum'], 1.0)
        res.append(r)
    return res


def main(files):
    for f in files:
        h, u, body = _rows(f)
        for v in body:
            d = dict(zip(h, v))
            un = dict(zip(h, u))
            line = [d['Kernel Name'][:60]]
            for k, n in KEYS:
                x = float(d[k].replace(',', ''))
                if k == 'gpu__time_duration.sum':
                    x *= _TIME.get(un[k], 1.0)
                if k.startswith('dram'):
                    x *= _BYTES.get(un[k], 1.0) / 1e6
                line.append(f"{n}={x:.1f}")
            st = sorted(((float(d[n].replace(',', '')), n.replace('smsp__pcsamp_warps_issue_stalled_', '')) for n in d
                         if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued')),
                        reverse=True)[:4]
            tot = sum(float(d[n].replace(',', '')) for n in d
                      if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued'))
            line.append("stalls: " + ", ".join(f"{n} {x / tot:.2f}" for x, n in st))
            print(f"{f.split('/')[-1]}: " + " ".join(line))


if __name__ == "__main__":
    main(sys.argv[1:])
