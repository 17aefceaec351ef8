"""Summarise ncu outputs for profiles/: launch-list CSV (per-kernel share) and --set full reports."""
import collections, csv, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers']


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
    h = rows[hi]
    ik, im, iv, iid = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        nm = r[ik].split('(')[0].replace('void ', '').replace('se::k::<unnamed>::', '')
        names[r[iid]] = nm
        per[nm][r[im]] += float(r[iv].replace(',', ''))
    cnt = collections.Counter(names.values())
    tot = sum(p['gpu__time_duration.sum'] for p in per.values())
    print(f"| kernel | launches | time share | avg us | DRAM MB/launch | DRAM GB/s |\n|---|---|---|---|---|---|")
    for nm in sorted(per, key=lambda n: -per[n]['gpu__time_duration.sum']):
        t = per[nm]['gpu__time_duration.sum']
        b = per[nm]['dram__bytes_read.sum'] + per[nm]['dram__bytes_write.sum']
        c = cnt[nm]
        print(f"| {nm} | {c} | {100*t/tot:.1f}% | {t/c/1e3:.2f} | {b/c/1e6:.2f} | {b/t:.0f} |")


def full(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"#### {d.get('Kernel Name', '')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"- {k}: {d[k]} {units[h.index(k)]}")


if __name__ == '__main__':
    (launches if sys.argv[1] == 'launches' else full)(sys.argv[2])
