"""Top SASS instructions by warp-stall samples from an ncu report:
python tools/ncu_hot.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
print("total samples", tot)
for r in rows[:n]:
    print(f'{int(r["Warp Stall Sampling (All Samples)"]):6d} {r["Address"][-5:]} {r["Source"].strip()[:90]}')
