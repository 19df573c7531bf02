"""Parse the ncu CSV of tools/probe_weights.py into profiles/fp64_weights.json."""
import csv
import json
import sys
from collections import defaultdict

path, out = sys.argv[1], sys.argv[2]
THREADS, REPS = 128 * 148, 64
rows = []
with open(path) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for r in csv.DictReader(lines):
    rows.append(r)
per = defaultdict(dict)
order = []
for r in rows:
    if "k_unary" not in r.get("Kernel Name", ""):
        continue
    key = r["ID"]
    if key not in order:
        order.append(key)
    per[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
names = ["exp", "log", "div"]
res = {"source": "ncu SASS op counts of tools/fp64probe.cu k_unary (64 calls/thread)",
       "formula": "2*dfma + dadd + dmul per call, minus the loop's 2 dadd"}
for nm, key in zip(names, order[:3]):
    m = per[key]
    dfma = m.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
    dadd = m.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
    dmul = m.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
    calls = THREADS * REPS
    res[nm] = round((2 * dfma + dadd + dmul) / calls - 2.0, 3)
    res[nm + "_raw"] = {"dfma": dfma / calls, "dadd": dadd / calls, "dmul": dmul / calls}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
