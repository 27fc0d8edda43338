"""Warp-stall samples of one kernel in an ncu report, aggregated per CUDA source line
(SASS offsets mapped to lines with nvdisasm -g on the cubin of the same build).
usage: ncu_lines.py REPORT KERNEL_REGEX MANGLED_NAME [N]
NCU_COL="Instructions Executed" aggregates executed warp instructions instead of stall samples;
WCSP_LIB names the build the report was captured with."""
import csv
import collections
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, mangled = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
so = os.environ.get("WCSP_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1511_06441_b200", "libwcsp.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
cubin = os.path.join(tmp, [f for f in os.listdir(tmp) if f.endswith(".cubin")][0])
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
start = dis.find(".text." + mangled + ":")
end = dis.find("\n.text.", start + 10) if start >= 0 else -1
dis = dis[start:end if end > 0 else None] if start >= 0 else ""
line_of, cur = {}, None
for l in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
i_s = hdr.index(os.environ.get("NCU_COL", "Warp Stall Sampling (All Samples)"))
items = [(int(r[0], 16), int(r[i_s])) for r in rows if len(r) == len(hdr) and r[0].startswith("0x") and r[i_s].isdigit()]
base = min(a for a, _ in items)
agg = collections.Counter()
seen = set()
for a, s in items:
    if a in seen:
        continue
    seen.add(a)
    agg[line_of.get(a - base, ("?", 0))] += s
tot = sum(agg.values()) or 1
src_cache = {}
def text(f, ln):
    p = os.path.join(os.path.dirname(so), "csrc", f)
    if p not in src_cache:
        src_cache[p] = open(p).read().splitlines() if os.path.exists(p) else []
    L = src_cache[p]
    return L[ln - 1].strip()[:90] if 0 < ln <= len(L) else ""
print(f"{kern}: {tot} samples, {len(line_of)} mapped instructions")
for (f, ln), s in agg.most_common(n):
    print(f"{100 * s / tot:5.1f}%  {f}:{ln}  {text(f, ln)}")
