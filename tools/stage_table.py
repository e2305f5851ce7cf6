"""Per-stage roofline table from an ncu launch list of one pipeline run
(metrics: gpu__time_duration, dram bytes, FP32/FP64 pipe, issue, smem
wavefronts and bank conflicts).  Percentages are time-weighted over the
launches of a kernel.
    python tools/stage_table.py gpurun_out/stagesx_c2.csv [hbm_peak_GBps]
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
per = OrderedDict()
for r in csv.DictReader(io.StringIO(txt)):
    d = per.setdefault((r["ID"], r["Kernel Name"]), {})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3,
          "msecond": 1e6}.get(unit, 1)
    d[r["Metric Name"]] = v
agg = OrderedDict()
total = 0.0
for (i, name), d in per.items():
    short = re.sub(r"\(.*", "", name.split("<")[0].split("::")[-1])
    m = re.search(r"<\(int\)(\d+)", name)
    if "sweep" in short and m:
        short += f"<b={m.group(1)}>"
    t = d.get("gpu__time_duration.sum", 0.0)
    a = agg.setdefault(short, dict(n=0, t=0.0, b=0.0, fma=0.0, f64=0.0, iss=0.0, wf=0.0, bc=0.0))
    a["n"] += 1
    a["t"] += t
    a["b"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    a["fma"] += t * d.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0)
    a["f64"] += t * d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0)
    a["iss"] += t * d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)
    a["wf"] += d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0)
    a["bc"] += d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 0)
    total += t
print("| kernel | launches | time (us) | share | DRAM | GB/s | HBM frac | FP32 pipe | FP64 pipe "
      "| issue | smem conflicts |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
    t = a["t"]
    gbs = a["b"] / t if t else 0.0
    conf = a["bc"] / a["wf"] if a["wf"] else 0.0
    print(f"| `{k}` | {a['n']} | {t/1e3:.1f} | {t/total:.1%} | {a['b']/1e6:.1f} MB | {gbs:.0f} "
          f"| {gbs/peak:.2f} | {a['fma']/t:.0f}% | {a['f64']/t:.0f}% | {a['iss']/t:.0f}% "
          f"| {conf:.1%} of {a['wf']/1e6:.1f}M wavefronts |")
print(f"\nTotal kernel time {total/1e3:.1f} us (ncu launch list: serialised, cold caches; "
      f"HBM peak {peak:.0f} GB/s from MEASURED_PEAKS.json).")
