"""Region summary of an `ncu --page source --csv` SASS export: per address range, executed warp
instructions, stall samples and the dominant stall reasons.
    python tools/sass_stalls.py gpurun_out/x/source.csv [n_top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    data.append((int(r[0], 16), r[1].strip(), int(r[ix["# Samples"]]), int(r[ix["Instructions Executed"]]),
                 {c: int(r[ix[c]]) for c in stall_cols}, int(r[ix["L1 Wavefronts Shared"]] or 0)))
base = data[0][0]
tot_s = sum(d[2] for d in data)
tot_i = sum(d[3] for d in data)
print(f"total samples {tot_s}, warp instructions {tot_i}, smem wavefronts {sum(d[5] for d in data)}")
agg = {}
for d in data:
    for c, v in d[4].items():
        agg[c] = agg.get(c, 0) + v
print("stall mix:", {k: round(v / tot_s, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("top instructions by samples:")
for d in sorted(data, key=lambda d: -d[2])[:n]:
    top = sorted(d[4].items(), key=lambda kv: -kv[1])[:2]
    print(f"  {d[0] - base:#07x} {d[2] / tot_s:6.2%} exec {d[3]:>10} {d[1][:60]:60s} {top}")
