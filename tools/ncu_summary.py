"""One-line ncu summaries (time, DRAM bytes, occupancy, issue, FP64 pipe, smem wavefronts, top stalls)
per kernel of .ncu-rep files: python tools/ncu_summary.py a.ncu-rep [...]"""
import csv, subprocess, sys
keys = [('gpu__time_duration.sum', 't_us'), ('dram__bytes_read.sum', 'dramR_MB'), ('dram__bytes_write.sum', 'dramW_MB'),
        ('sm__warps_active.avg.pct_of_peak_sustained_active', 'warps%'), ('smsp__issue_active.avg.pct_of_peak_sustained_active', 'issue%'),
        ('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'fp64%'),
        ('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed', 'smem_wf%'),
        ('launch__registers_per_thread', 'regs')]
for f in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', f, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v)); un = dict(zip(h, u))
        line = [d['Kernel Name'][:60]]
        for k, n in keys:
            x = float(d[k].replace(',', ''))
            if k == 'gpu__time_duration.sum' and un[k] == 'msecond': x *= 1e3
            if k.startswith('dram') and un[k] == 'Gbyte': x *= 1e3
            line.append(f"{n}={x:.1f}")
        st = sorted(((float(d[n].replace(',', '')), n.replace('smsp__pcsamp_warps_issue_stalled_', '')) for n in d
                     if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued')), reverse=True)[:4]
        tot = sum(float(d[n].replace(',', '')) for n in d if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued'))
        line.append("stalls: " + ", ".join(f"{n} {x / tot:.2f}" for x, n in st))
        print(f"{f.split('/')[-1]}: " + " ".join(line))
