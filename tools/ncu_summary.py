"""Summarise an ncu --set full report into markdown (for profiles/).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep "title" > profiles/x.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-instr"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instr"),
    ("smsp__inst_executed.sum", "warp-instr executed"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed", "smem load wavefronts % peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# {title}\n")
    print(f"Source: `{path}` (ncu --set full --clock-control none --import-source on).\n")
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## `{name[:120]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"| {label} (`{key}`) | {vals[i]} | {units[i]} |")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    st.append((float(vals[i].replace(",", "")), h))
                except ValueError:
                    pass
        print("\nTop warp stall reasons (cycles per issued instruction):\n")
        for v, h in sorted(st, reverse=True)[:8]:
            short = h.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", "")
            print(f"* {short}: {v:.3f}")
        print()


def source_lines(path, top=25):
    """Per-source-line share of executed warp instructions and of the warp
    stall samples (ncu --page source --print-source cuda,sass)."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    cur, hdr, res = None, None, {}

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[0] == "":
            continue
        res[(cur, num(r[0]))] = (num(r[7]), num(r[4]), r[1].strip()[:90])
    tot = sum(v[0] for v in res.values()) or 1
    ts = sum(v[1] for v in res.values()) or 1
    print(f"Top source lines by executed warp instructions ({tot} total; stall samples {ts}):\n")
    print("| file:line | instr share | stall-sample share | source |\n|---|---|---|---|")
    for (f, ln), (ni, ns, src) in sorted(res.items(), key=lambda x: -x[1][0])[:top]:
        src = src.replace("|", "\\|")
        print(f"| {f}:{ln} | {100 * ni / tot:.1f}% | {100 * ns / ts:.1f}% | `{src}` |")
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
    if "--lines" in sys.argv:
        source_lines(sys.argv[1])
