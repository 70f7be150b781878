"""Summarise an ncu source page (SASS) by stall samples.

    python tools/ncu_source.py REP KERNEL_REGEX [TOP] [--regions]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Address":
        break                      # the listing repeats per captured launch
    if len(r) > 5:
        data.append(r)
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")


def val(r):
    try:
        return int(r[i_s])
    except ValueError:
        return 0


tot = sum(val(r) for r in data) or 1
print("instructions", len(data), "samples", tot)
if "--regions" in sys.argv:
    step = 100
    for k in range(0, len(data), step):
        s = sum(val(r) for r in data[k:k + step])
        if s:
            print(f"  [{k:5d}..] {s:6d} {100 * s / tot:5.1f}%  {data[k][i_src].strip()[:60]}")
ranked = sorted(range(len(data)), key=lambda k: -val(data[k]))[:top]
for k in sorted(ranked):
    print(f"{k:5d} {val(data[k]):6d} {100 * val(data[k]) / tot:5.1f}%  {data[k][i_src].strip()[:90]}")
