"""Print the headline numbers of a bench.py JSON line (file argument)."""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]).read().splitlines() if ln.strip().startswith("{")][-1])
print("value", round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 2), "launches", d.get("gpu_launches"),
      "clocks", d.get("clocks"))
for p in d.get("points", []):
    print(f"  {p['point']:28s} {p.get('gflops', 0):10.1f} GF/s  frac {p['roofline_frac']:.3f}  {p['ms']:8.3f} ms")
r = d.get("roofline")
if r:
    print("roofline", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
for key in ("e2e", "cpu_baseline"):
    if d.get(key):
        print(key, {k: v for k, v in d[key].items() if k not in ("sample", "per_point_gflops", "per_point_gflops_1core")})
if d.get("inplace"):
    ip = d["inplace"]
    print("inplace", round(ip["value"], 1), [(p["point"], round(p["roofline_frac"], 3), round(p["ms"], 2)) for p in ip["points"]])
if d.get("gemm"):
    g = d["gemm"]
    print("gemm c1", round(g["c1"]["gflops"], 1), round(g["c1"]["roofline_frac"], 3), "c3", round(g["c3"]["value"], 1),
          g["c3"]["frac_n_ge_64"], g["c3"]["frac_n_le_16"], round(g["c3"]["sweep_ms"], 1))
    print("  c3 low:", [(p["point"].split()[1], round(p["roofline_frac"], 2)) for p in g["c3"]["points"]
                        if p["roofline_frac"] < 0.6])
