"""Implemented FP32 work and DRAM traffic of the level-0 sweep, from ncu.

    python tools/flop_check.py capture OUT.json [C1 C2 ...]   # on the GPU box
    python tools/flop_check.py show OUT.json

`capture` runs tools/prof_once.py for each config under
    ncu --metrics <time, dram bytes, FP32 thread-instruction counts>
restricted to the level-0 sweep kernels (sweep4_kernel + prior_select_kernel
on sweep4 levels; sweep2_kernel otherwise) and records, per config, every
matching launch.  FP32 flops = FADD + FMUL + 2 x FFMA thread instructions
(predicated-on), the implemented count SURVEY 8(d) asks a sliding-sum design
to declare.  bench.py reads the committed JSON (profiles/) for the roofline's
`achieved` numerator and `traffic`.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
        "usecond": 1.0, "msecond": 1e3, "inst": 1, "": 1}


def capture(out, cfgs):
    res = {}
    for c in cfgs:
        log = os.path.join(ROOT, "gpurun_out", f"flops_{c}.csv")
        cmd = ["ncu", "--clock-control", "none", "--metrics", ",".join(METRICS),
               "-k", "regex:sweep4_kernel|prior_select_kernel|sweep2_kernel", "--csv",
               "--log-file", log, sys.executable, os.path.join(ROOT, "tools", "prof_once.py"), c]
        subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
        txt = open(log).read()
        txt = txt[txt.index('"ID"'):]
        launches = {}
        for r in csv.DictReader(io.StringIO(txt)):
            d = launches.setdefault(r["ID"], {"kernel": r["Kernel Name"]})
            v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
            d[r["Metric Name"]] = v
        res[c] = list(launches.values())
    json.dump(res, open(out, "w"), indent=1)


def summary(rec):
    """Level-0 sweep of one config: the last sweep4 launch (+ its
    prior_select), else the last sweep2 launch (levels run coarse to fine)."""
    s4 = [l for l in rec if "sweep4_kernel" in l["kernel"]]
    ps = [l for l in rec if "prior_select_kernel" in l["kernel"]]
    main = s4[-1] if s4 else [l for l in rec if "sweep2_kernel" in l["kernel"]][-1]

    def fl(l):
        return (2 * l["smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"]
                + l["smsp__sass_thread_inst_executed_op_fadd_pred_on.sum"]
                + l["smsp__sass_thread_inst_executed_op_fmul_pred_on.sum"])
    out = {"kernel": main["kernel"].split("(")[0], "flops": fl(main),
           "us": main["gpu__time_duration.sum"],
           "dram_bytes": main["dram__bytes_read.sum"] + main["dram__bytes_write.sum"]}
    if s4 and ps:
        out["prior_select"] = {"flops": fl(ps[-1]), "us": ps[-1]["gpu__time_duration.sum"],
                               "dram_bytes": ps[-1]["dram__bytes_read.sum"]
                               + ps[-1]["dram__bytes_write.sum"]}
    return out


if __name__ == "__main__":
    if sys.argv[1] == "capture":
        capture(sys.argv[2], sys.argv[3:] or ["C1", "C2", "C3", "C4", "C5"])
    else:
        for c, rec in json.load(open(sys.argv[2])).items():
            s = summary(rec)
            print(c, json.dumps(s))
