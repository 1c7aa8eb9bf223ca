"""Summarise an ncu report per CUDA source line of generator_tc.cu (stall samples,
executed instructions).  Usage: python tests/ncu_lines.py report.ncu-rep cubin [N]"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep, cubin = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if l.startswith(".text._ZN4mgsr2tc8k_gen_tc")][0]
cur = None; off2line = {}
for l in dis[start:]:
    m = re.search(r'generator_tc.cu", line (\d+)', l)
    if m: cur = int(m.group(1))
    m2 = re.match(r"\s+/\*([0-9a-f]{4,6})\*/", l)
    if m2: off2line[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); hdr = rows[1]; data = rows[2:]
iss = hdr.index("Warp Stall Sampling (All Samples)"); iex = hdr.index("Instructions Executed")
agg = defaultdict(lambda: [0, 0])
for i, r in enumerate(data):
    ln = off2line.get(i * 16)
    agg[ln][0] += int(r[iss] or 0); agg[ln][1] += int(r[iex] or 0)
tot = sum(v[0] for v in agg.values()); totex = sum(v[1] for v in agg.values())
src = open("paper_2403_07936_b200/csrc/generator_tc.cu").read().split("\n")
for ln, (s, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{str(ln):>5} {100*s/tot:5.1f}% ex {100*ex/totex:5.1f}%  {src[ln-1].strip()[:80] if ln else '?'}")
