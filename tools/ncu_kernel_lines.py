"""Per-source-line instruction and stall-sample totals of ONE kernel of an
ncu report: python tools/ncu_kernel_lines.py report.ncu-rep kernel-regex [n]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
rows, hdr, fname = [], None, None
for l in out.splitlines():
    if l.startswith('"File Path"'):
        fname = l.split(",", 1)[1].strip('"').rsplit("/", 1)[-1]
        continue
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        continue
    if hdr is None or not l.startswith('"'):
        continue
    r = next(csv.reader([l]))
    if len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    rows.append((fname, int(r[0]), r[1].strip()[:90], int(d["Instructions Executed"] or 0),
                 int(d["Warp Stall Sampling (All Samples)"] or 0)))
tot = sum(x[4] for x in rows) or 1
print("samples", tot, "instructions", sum(x[3] for x in rows))
for x in sorted(rows, key=lambda x: -x[4])[:n]:
    print("%5.1f%% %9d %-14s %5d %s" % (100 * x[4] / tot, x[3], x[0], x[1], x[2]))
