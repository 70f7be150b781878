"""Summarise a round's ncu evidence into profiles/ (tracked).

    python tools/summarize_ncu.py ROUND LAUNCHES_CSV FULL_REP [WORKLOAD]

Writes profiles/<ROUND>_launches.md (per-kernel share of one solve from the
serialised, cold-cache launch list), profiles/<ROUND>_ncu_full.md (key
metrics + top stall reasons per captured kernel) and
profiles/ncu_traffic_<ROUND>_<WORKLOAD>.json (dram bytes and L2 sectors per
launch of the same workload, read by bench.py for roofline.traffic).
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

rnd, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else "cfg2"
out = Path(__file__).resolve().parents[1] / "profiles"
out.mkdir(exist_ok=True)

# bench.py names -> kernel names
BENCH_NAME = {"k_xt_coop": "xt", "k_segsum<0>": "spmv_rows", "k_segsum<1>": "smoother",
              "k_cg_step": "cg_step", "k_shift_update": "shift_update",
              "k_spmm_scores": "spmm_scores", "k_combine_basis": "combine_basis"}


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("fsda::", "")
    # templated kernels: k_segsum<0, fsda::SegArgsT<double, double>> -> k_segsum<0>
    if n.startswith("k_segsum<"):
        n = "k_segsum<" + n[len("k_segsum<")] + ">"
    elif "<" in n:
        n = n.split("<")[0]
    return n


rows = [r for r in csv.reader(open(launches)) if len(r) > 10 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    k = short(r[4])
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
lines = [f"# {rnd}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
         f"One eager {workload} solve (FSDA_B200_EAGER=1, tools/ncu_solve.py --solves 1), including the",
         "upload (CSC sort, plans).  Serialised and cold-cache: compare shares, not absolutes.", "",
         "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| `{k}` | {n} | {t / n / 1e3:.2f} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
(out / f"{rnd}_launches.md").write_text("\n".join(lines) + "\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr = r[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum"]
units = r[1] if len(r) > 1 else []
md = [f"# {rnd}: ncu --set full (one captured launch per kernel, iteration 2 of a {workload} solve)", ""]
traffic = {}
for row in r[2:]:
    name = short(row[hdr.index("Kernel Name")])
    md.append(f"## `{name}`")
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            md.append(f"- {k}: {row[i]} {units[i] if units else ''}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                v = float(row[i])
            except ValueError:
                continue
            if v > 0:
                stalls.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    stalls.sort(reverse=True)
    tot_s = sum(v for v, _ in stalls) or 1
    md.append("- top stalls: " + ", ".join(f"{n} {100 * v / tot_s:.0f}%" for v, n in stalls[:5]))
    md.append("")

    def mb(k):
        i = hdr.index(k)
        v = float(row[i])
        u = units[i] if units else "byte"
        return v * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)

    bench = BENCH_NAME.get(name)
    if bench:
        ent = {"kernel": name, "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")}
        for k in ("lts__t_sectors.sum", "lts__t_sectors_srcunit_tex_op_read.sum"):
            if k in hdr:
                try:
                    ent["l2_sectors_per_launch" if k == "lts__t_sectors.sum" else "l2_read_sectors_per_launch"] = \
                        float(row[hdr.index(k)])
                except ValueError:
                    pass
        traffic[bench] = ent
(out / f"{rnd}_ncu_full.md").write_text("\n".join(md) + "\n")
(out / f"ncu_traffic_{rnd}_{workload}.json").write_text(
    json.dumps({"round": rnd, "workload": workload, "kernels": traffic}, indent=1))
print("\n".join(lines))
print(json.dumps(traffic, indent=1))
