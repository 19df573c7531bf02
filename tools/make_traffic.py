"""profiles/traffic.json: DRAM bytes (read + write) per launch of each kernel,
from `ncu --set full` captures taken at the bench's own problem sizes
(tools/gpu_check.sh).  bench.py reports it as roofline.traffic."""
import json
import sys

sys.path.insert(0, "tools")
from ncu_summary import summarise  # noqa: E402

out = {"_source": "ncu --set full --clock-control none (dram__bytes_read.sum + dram__bytes_write.sum)",
       "_captures": {}}
for name, rep in [("k_besselj", "gpurun_out/prof_bessel.ncu-rep"),
                  ("k_ba_jac", "gpurun_out/prof_ba.ncu-rep"),
                  ("k_gmm", "gpurun_out/prof_gmm.ncu-rep")]:
    try:
        rows = summarise(rep)
    except Exception as err:  # noqa: BLE001
        print("skip", rep, err)
        continue
    for r in rows:
        kn = r["kernel"].split("(")[0].replace("void ", "").strip()
        b = (r.get("dram_read_MB", 0) + r.get("dram_write_MB", 0)) * 1e6
        out.setdefault(kn, round(b))
        out["_captures"][kn] = rep
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
