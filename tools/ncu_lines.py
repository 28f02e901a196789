"""Stall samples per CUDA source line from an ncu report (run here, no GPU).

    python tools/ncu_lines.py <rep.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg, tot, fname = {}, 0, ""
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    if len(r) < 5 or not r[0].isdigit():
        continue
    try:
        v = int(r[4])
    except ValueError:
        continue
    key = (fname, int(r[0]), r[1][:80])
    agg[key] = agg.get(key, 0) + v
    tot += v
print(rep, "samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {k[0]}:{k[1]}  {k[2]}")
