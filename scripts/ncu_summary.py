"""Summarise ncu reports / launch lists for profiles/ (run here, no GPU)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_atom.sum',
        'lts__t_sectors_srcunit_tex_op_write.sum', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'sm__inst_executed.avg.per_cycle_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("=====", r[h.index("Kernel Name")][:40])
        items = []
        for i, name in enumerate(h):
            if "smsp__pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
                try:
                    items.append((float(r[i].replace(",", "")), name[33:]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items) or 1
        print("  stalls:", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(items, reverse=True)[:6]))
        for k in KEYS:
            if k in h:
                print(f"  {k} = {r[h.index(k)]} {units[h.index(k)]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ni, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        n = r[ni].split("(")[0]
        tot[n] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[n] += 1
    s = sum(tot.values())
    for n in sorted(tot, key=lambda x: -tot[x]):
        print(f"  {n[:50]:50s} {cnt[n]:6d} launches {tot[n] / 1e3:10.3f} ms {100 * tot[n] / s:5.1f}%")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("#", p)
        report(p) if p.endswith(".ncu-rep") else launches(p)
