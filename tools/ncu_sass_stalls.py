"""Hottest SASS instructions of one kernel of an ncu report with their stall
reasons: python tools/ncu_sass_stalls.py report.ncu-rep kernel-regex [n]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
recs = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "Address"]
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in recs) or 1
recs.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
for r in recs[:n]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((int(r[h] or 0), h[6:]) for h in st), reverse=True)[:3]
    print("%5.1f%% %-60s %s" % (100 * s / tot, r["Source"][:60],
                                " ".join(f"{k}:{v}" for v, k in top if v)))
