"""Per-kernel HBM roofline table from an ncu launch list with
gpu__time_duration / dram__bytes_read / dram__bytes_write (one pipeline run).
    python tools/stage_table.py gpurun_out/stages_c2.csv [peak_GBps]
"""
import csv
import io
import re
import sys
from collections import OrderedDict

path = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6552.0
txt = open(path).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
per = OrderedDict()
for r in rows:
    k = (r["ID"], r["Kernel Name"])
    d = per.setdefault(k, {})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    if r["Metric Name"].startswith("dram"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    elif unit == "usecond":
        v *= 1e3
    elif unit == "msecond":
        v *= 1e6
    d[r["Metric Name"]] = v
agg = OrderedDict()
total = 0.0
for (i, name), d in per.items():
    short = re.sub(r"\(.*", "", name.split("<")[0].split("::")[-1])
    m = re.search(r"<\(int\)(\d+)", name)
    if "sweep" in short and m:
        short += f"<b={m.group(1)}>"
    a = agg.setdefault(short, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    total += d.get("gpu__time_duration.sum", 0)
print(f"| kernel | launches | time (us) | share | DRAM bytes | achieved GB/s | HBM frac |")
print("|---|---|---|---|---|---|---|")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    gbs = b / t if t else 0
    print(f"| `{k}` | {n} | {t/1e3:.1f} | {t/total:.1%} | {b/1e6:.1f} MB | {gbs:.0f} | {gbs/peak:.2f} |")
print(f"\ntotal kernel time {total/1e3:.1f} us (serialised, cold-cache launch list)")
