"""Per-source-line stall samples and instruction counts of one kernel in an
ncu report: maps the report's SASS page onto source lines through the line
table of the locally built object (nvdisasm -g), since this ncu prints no
metrics on its CUDA source page.
Usage: python tools/ncu_lines.py REPORT.ncu-rep OBJECT.o KERNEL_SUBSTRING [top=30]"""
import collections
import csv
import re
import subprocess
import sys
import tempfile
from pathlib import Path

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ai, si, ci = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(data[0][ai], 16)
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, capture_output=True)
    cub = next(Path(td).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout.split("\n")
# locate the kernel (mangled name containing kname and matching instruction count)
funcs, cur, lines, line = {}, None, None, None
for l in sass:
    m = re.match(r"^\s*\.text\.(\S+):", l) or re.match(r"^(_Z\S+):$", l.strip())
    if l.startswith(".text."):
        cur = l[len(".text."):].rstrip(":")
        funcs[cur] = {}
        line = None
        continue
    m = re.search(r'//## File ".*", line (\d+)', l)
    if m:
        line = int(m.group(1))
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
    if m and cur is not None:
        funcs[cur][int(m.group(1), 16)] = line
cands = [f for f in funcs if kname in f and len(funcs[f]) >= len(data) - 8]
cands.sort(key=lambda f: abs(len(funcs[f]) - len(data)))
fmap = funcs[cands[0]]
print("kernel:", cands[0][:120], "sass rows", len(data), "map", len(fmap))
samp, ins = collections.Counter(), collections.Counter()
for r in data:
    off = int(r[ai], 16) - base
    ln = fmap.get(off)
    samp[ln] += float(r[si] or 0)
    ins[ln] += float(r[ci] or 0)
ts, ti = sum(samp.values()), sum(ins.values())
src = Path(sys.argv[5]).read_text().split("\n") if len(sys.argv) > 5 else None
for ln, s in samp.most_common(top):
    txt = src[ln - 1].strip()[:80] if src and ln else ""
    print(f"{ln}\t{100 * s / ts:5.1f}% smp\t{100 * ins[ln] / ti:5.1f}% ins\t{txt}")
