import json, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log"
l = [x for x in open(path) if x.startswith("{")][-1]
d = json.loads(l)
print("value", round(d["value"], 2), "ms/step", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"], 2),
      "launches", d.get("gpu_launches"))
r = d.get("roofline")
if r:
    print("top", r["kernel"], round(r["achieved"], 1), "GB/s frac", round(r["frac"], 3), "share", round(r["share_of_step"], 3))
    for k, v in r["kernels"].items():
        print(f"  {k:16s} {v}")
print("pair", d.get("spmv_pair"))
print("cpu", d.get("cpu_baseline", {}) and d["cpu_baseline"].get("value"), d.get("clocks"))
