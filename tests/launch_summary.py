"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) of
``bench.py`` into per-kernel totals and shares of one V-cycle step.

    python tests/launch_summary.py launches.csv steps out.json
"""
import csv
import io
import json
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = re.sub(r"^void ", "", name)
    return name


def main():
    path, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    rows = [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    # only our kernels (mgsr namespace / C-ABI translation units) belong to the step
    ours = [r for r in rows if "mgsr::" in r["Kernel Name"] or "tc::" in r["Kernel Name"]]
    agg = defaultdict(lambda: [0, 0.0])
    for r in ours:
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
    total = sum(v[1] for v in agg.values())
    kern = {k: {"launches": n, "us_total": round(us, 1), "share": round(us / total, 4)}
            for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    res = {"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none, cold-cache serialised "
           "launches (MGSR_NO_GRAPH=1 eager issue of the graph's kernel sequence); warmup+timed steps all listed",
           "all_launches": len(rows), "mgsr_launches": len(ours), "mgsr_us_total": round(total, 1),
           "kernels": kern}
    json.dump(res, open(out, "w"), indent=1)
    for k, v in kern.items():
        print(f"{v['share']*100:6.2f}% {v['us_total']:10.1f} us  x{v['launches']:4d}  {k[:90]}")


if __name__ == "__main__":
    main()
