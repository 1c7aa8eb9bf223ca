"""Summarise an ncu report per CUDA source line (stall samples, executed
instructions) by mapping SASS offsets through nvdisasm line info.

    python tests/ncu_lines.py report.ncu-rep object.o [N] [kernel-substring] [source.cu]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, obj = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
kern = sys.argv[4] if len(sys.argv) > 4 else "k_gen_tc"
srcname = sys.argv[5] if len(sys.argv) > 5 else "generator_tc.cu"
cubin = obj
if obj.endswith(".o"):
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd="/tmp", capture_output=True)
    import glob
    cands = sorted(glob.glob("/tmp/*.sm_100a.cubin"), key=lambda p: -__import__("os").path.getmtime(p))
    cubin = cands[0]
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout.split("\n")
rep_name = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
starts = [i for i, l in enumerate(dis) if l.startswith(".text.") and kern in l]
# pick the function ncu profiled: match mangled template args roughly by first hit
start = starts[0]
cur = None
off2line = {}
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(re.escape(srcname) + r'", line (\d+)', l)
    if m:
        cur = int(m.group(1))
    m2 = re.match(r"\s+/\*([0-9a-f]{4,6})\*/", l)
    if m2:
        off2line[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
iss = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
agg = defaultdict(lambda: [0, 0])
for i, r in enumerate(data):
    ln = off2line.get(i * 16)
    agg[ln][0] += int(r[iss] or 0)
    agg[ln][1] += int(r[iex] or 0)
tot = sum(v[0] for v in agg.values()) or 1
totex = sum(v[1] for v in agg.values()) or 1
src = open(f"paper_2403_07936_b200/csrc/{srcname}").read().split("\n")
for ln, (s, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{str(ln):>5} stall {100*s/tot:5.1f}% ex {100*ex/totex:5.1f}%  {src[ln-1].strip()[:80] if ln else '?'}")
