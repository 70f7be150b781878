"""Stall samples per CUDA source line (needs a report captured with
--import-source on and a -lineinfo build).

    python tools/ncu_lines.py REP KERNEL_REGEX [TOP]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
func = sys.argv[4] if len(sys.argv) > 4 else None   # substring of the function name
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
samples = defaultdict(int)
text = {}
fname = "?"
cur = None
i_s = None
seen = set()
skip = False
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Function Name":
        skip = func is not None and func not in r[1]
        continue
    if func is not None and skip:
        continue
    if r[0] == "Line No":
        i_s = r.index("Warp Stall Sampling (All Samples)")
        continue
    if i_s is None or len(r) <= i_s:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()
    else:
        addr = r[2]
        if (cur, addr) in seen:
            continue
        seen.add((cur, addr))
        try:
            samples[cur] += int(r[i_s])
        except ValueError:
            pass
tot = sum(samples.values()) or 1
print("samples", tot)
for k in sorted(samples, key=lambda k: -samples[k])[:top]:
    print(f"{k[0]}:{k[1]:5d} {samples[k]:6d} {100 * samples[k] / tot:5.1f}%  {text.get(k, '')[:90]}")
