"""Summarise ncu reports into profiles/ (launch-list shares + per-kernel key metrics)."""
import collections, csv, json, subprocess, sys

def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r); h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi: continue
        k = r[ki].split('(')[0].replace('void ', '').replace('gbxcu::', '')
        a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(',', ''))
    # bench.py's own pipe-peak probes (tools/peaks.cu) are not part of the step
    for probe in [k for k in agg if 'peak_kernel' in k]:
        agg.pop(probe)
    tot = sum(v[1] for v in agg.values())
    return [(k, c, t / c / 1e3, t / tot) for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__grid_size',
        'launch__registers_per_thread', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg']

def kernel_metrics(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]; res = []
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
        m = {'kernel': d.get('Kernel Name', '').split('(')[0]}
        for k in KEYS:
            if k in d and d[k] not in ('', 'n/a'):
                try:
                    v = float(d[k].replace(',', ''))
                    if u.get(k) in scale: v, k2 = v * scale[u[k]], k + ' [bytes]'
                    else: k2 = k + (f' [{u[k]}]' if u.get(k) else '')
                    m[k2] = v
                except ValueError: pass
        st = {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''): float(d[k])
              for k in hdr if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio') and d.get(k)}
        m['top_stalls'] = dict(sorted(st.items(), key=lambda x: -x[1])[:5])
        res.append(m)
    return res

if __name__ == '__main__':
    tag = sys.argv[1]
    lines = [f"# ncu summary {tag}", "", "## Launch list (bench.py --steps 1 --warmup 1; cold-cache, serialised)", "",
             "| kernel | launches | avg us | share |", "|---|---|---|---|"]
    shares = launch_shares('gpurun_out/launches.csv')
    for k, c, avg, sh in shares:
        lines.append(f"| {k} | {c} | {avg:.1f} | {sh:.1%} |")
    # the timed step of the headline (one fit epoch): every kernel of a
    # --no-secondary run (launches_step.csv) when present, else the fit kernels
    import os
    if os.path.exists('gpurun_out/launches_step.csv'):
        step = [(k, c, avg) for k, c, avg, _ in launch_shares('gpurun_out/launches_step.csv')]
    else:
        step = [(k, c, avg) for k, c, avg, _ in shares
                if k.startswith(('train_epoch', 'shuffle_epoch', 'iota_kernel', 'finish_epoch'))]
    tot = sum(c * avg for _, c, avg in step)
    lines += ["", "### Share of the headline step (bench.py --no-secondary: fit epochs only)", "",
              "| kernel | launches | avg us | share of step |", "|---|---|---|---|"]
    for k, c, avg in step:
        lines.append(f"| {k} | {c} | {avg:.1f} | {c * avg / tot:.1%} |")
    allm = []
    for rep in ['gpurun_out/prof_train.ncu-rep', 'gpurun_out/prof_other.ncu-rep']:
        try: allm += kernel_metrics(rep)
        except Exception as e: print('skip', rep, e)
    lines += ["", "## Full captures (--set full --clock-control none)", ""]
    for m in allm:
        lines.append(f"### {m['kernel']}")
        for k, v in m.items():
            if k != 'kernel': lines.append(f"- {k}: {v}")
        lines.append("")
    open(f'profiles/{tag}_ncu_summary.md', 'w').write("\n".join(lines) + "\n")
    json.dump(allm, open(f'profiles/{tag}_ncu_metrics.json', 'w'), indent=1)
    print("\n".join(lines[:40]))
