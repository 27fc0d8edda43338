"""Top SASS instructions by warp-stall samples for one kernel of an ncu report (with -lineinfo:
maps back to source lines via --print-source sass,cuda is not needed: we group by SASS)."""
import csv
import io
import subprocess
import sys

path, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
items = []
for r in rows:
    if len(r) == len(hdr) and r[0].startswith("0x"):
        try:
            items.append((int(r[i_s]), r[1].strip()))
        except ValueError:
            pass
tot = sum(s for s, _ in items) or 1
print(f"{kern}: {tot} samples")
for s, src in sorted(items, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  {src[:110]}")
