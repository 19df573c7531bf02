"""Summarise an ncu --set full report (raw page) into the metrics the roofline
needs: duration, DRAM bytes, pipe utilisation, issue, occupancy, top stalls.
usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6, "ns"),
    "dram_read_MB": ("dram__bytes_read.sum", None, None),
    "dram_write_MB": ("dram__bytes_write.sum", None, None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1, None),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1, None),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1, None),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1, None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1, None),
    "regs_per_thread": ("launch__registers_per_thread", 1, None),
    "threads_per_warp_active": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1, None),
    "inst_executed": ("smsp__inst_executed.sum", 1, None),
    "dfma": ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 1, None),
    "dadd": ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 1, None),
    "dmul": ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 1, None),
    "sm_clock_GHz": ("sm__cycles_elapsed.avg.per_second", 1, None),
}
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "barrier", "math_pipe_throttle",
          "not_selected", "mio_throttle", "lg_throttle", "no_instruction", "branch_resolving",
          "dispatch_stall", "tex_throttle", "membar", "drain", "sleeping", "selected"]


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def summarise(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, zip(units, vals)))
        rec = {"kernel": d.get("Kernel Name", ("", ""))[1][:90]}
        for name, (key, scale, _) in KEYS.items():
            if key not in d:
                continue
            unit, v = d[key]
            f = to_float(v)
            if f is None:
                continue
            if name.endswith("_MB"):
                f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
            elif name == "duration_ms":
                f = f * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1.0)
            elif name == "sm_clock_GHz":
                f = f * {"hz": 1e-9, "Ghz": 1.0, "Mhz": 1e-3}.get(unit, 1.0)
            rec[name] = round(f, 4)
        stalls = {}
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d:
                f = to_float(d[k][1])
                if f:
                    stalls[s] = round(f, 3)
        rec["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        if "dfma" in rec:
            rec["fp64_flops_executed"] = 2 * rec["dfma"] + rec.get("dadd", 0) + rec.get("dmul", 0)
        out.append(rec)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    for r in res:
        print(json.dumps(r))
