"""Per-CUDA-source-line warp-instruction and stall-sample totals of the
kernel in an ncu report (the cuda,sass source page lists every source line
with its totals): python tools/ncu_lines.py report.ncu-rep [n] [file-filter]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows, fname = [], None
hdr = None
for l in out.splitlines():
    if l.startswith('"File Path"'):
        fname = l.split(",", 1)[1].strip('"').rsplit("/", 1)[-1]
        continue
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        continue
    if hdr is None or not l.startswith('"') or l.startswith('""'):
        continue
    r = next(csv.reader([l]))
    if len(r) != len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        rows.append((fname, int(r[0]), r[1].strip(), int(d["Instructions Executed"] or 0),
                     int(d["Warp Stall Sampling (All Samples)"] or 0)))
    except ValueError:
        pass
ti = sum(x[3] for x in rows)
ts = sum(x[4] for x in rows)
print(f"total warp instructions {ti}, stall samples {ts}")
for key, nm in ((3, "instructions"), (4, "samples")):
    print(f"--- top lines by {nm}")
    for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[key])[:n]:
        print(f"{f}:{ln:<5d} {100 * ins / max(ti, 1):5.1f}% ins {100 * smp / max(ts, 1):5.1f}% smp  {src[:80]}")


def group(ranges):
    """Totals per named (file, lo, hi) line range."""
    res = {}
    for nm, (f, lo, hi) in ranges.items():
        sel = [x for x in rows if x[0] == f and lo <= x[1] <= hi]
        res[nm] = (sum(x[3] for x in sel), sum(x[4] for x in sel))
    return res


if len(sys.argv) > 3 and sys.argv[3] == "bessel":
    R = {"exp (fexp.cuh)": ("fexp.cuh", 1, 400), "rexp wrapper": ("besselj.cu", 120, 165),
         "logpair/logi": ("besselj.cu", 100, 110), "fwd_trip (pred tail)": ("besselj.cu", 185, 206),
         "rev_trip": ("besselj.cu", 207, 245), "prologue": ("besselj.cu", 262, 300),
         "fwd main loop": ("besselj.cu", 301, 420), "rev loops": ("besselj.cu", 421, 458),
         "epilogue": ("besselj.cu", 459, 495), "chunk/sort/store": ("besselj.cu", 720, 900)}
    g = group(R)
    other = ti - sum(v[0] for v in g.values())
    for nm, (i, s) in g.items():
        print(f"{nm:22s} {100 * i / ti:5.1f}% ins {100 * s / ts:5.1f}% smp")
    print(f"{'other':22s} {100 * other / ti:5.1f}% ins")
