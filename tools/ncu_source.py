"""Summarise an ncu source page (SASS) by stall samples: python tools/ncu_source.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i_s]) for r in data if r[i_s].isdigit())
print("total samples", tot)
for k, r in enumerate(data):
    pass
ranked = sorted(((int(r[i_s]), k, r[i_src]) for k, r in enumerate(data) if r[i_s].isdigit()), reverse=True)[:top]
for s, k, src in sorted(ranked, key=lambda x: x[1]):
    print(f"{k:5d} {s:6d} {100*s/tot:5.1f}%  {src.strip()[:90]}")
