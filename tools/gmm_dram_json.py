"""profiles/r02/gmm_c3_dram_per_eval.json from gpurun_out/gmm_dram_eval.csv
(tools/gpu_gmm_dram.sh): the last evaluation's kernels."""
import csv
import json

rows = [r for r in csv.reader(open("gpurun_out/gmm_dram_eval.csv")) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ids = hdr.index("ID")
per = {}
recs = rows[1:]
# one evaluation = the last len(kernels) launches
names = []
for r in recs:
    if r[ki] not in names:
        names.append(r[ki])
last_ids = sorted({int(r[ids]) for r in recs})[-len(names):]
for r in recs:
    if int(r[ids]) not in last_ids:
        continue
    key = r[ki][:32]
    v = float(r[vi].replace(",", "")) / 1e6
    unit_scale = 1.0
    per.setdefault(key, [0.0, 0.0])
    per[key][0 if "read" in r[mi] else 1] += v * unit_scale
tot = sum(a + b for a, b in per.values())
out = {"what": "DRAM MB per kernel of ONE drop-in configs[2] GMM evaluation: L2 evicted before "
               "the evaluation by READING 256 MiB (clean lines, no write-back lands in the "
               "counters), no cache flush between the evaluation's kernels (ncu --cache-control "
               "none); tools/gpu_gmm_dram.sh",
       "per_kernel_read_write_MB": {k: [round(a, 3), round(b, 3)] for k, (a, b) in per.items()},
       "total_MB": round(tot, 2),
       "algorithmic_MB": "x 5.12 + parameters in / gradient out ~0.9"}
json.dump(out, open("profiles/r02/gmm_c3_dram_per_eval.json", "w"), indent=1)
print(json.dumps(out, indent=1))
