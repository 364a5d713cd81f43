"""Print the markdown tables of profiles/r02_summary.md / README from the bench lines in profiles/."""
import json, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
names = {1: "cfg1 random COO 1000^2", 2: "cfg2 2D FEM N = 1000", 3: "cfg3 3D FEM 100^3", 4: "cfg4 heavy-duplicate", 5: "cfg5 2D FEM N = 8000"}
print("| config | L | ms / step | G triplets/s | path roofline | dominant kernel (frac of peak) | e2e ms |")
print("|---|---|---|---|---|---|---|")
for c in (1, 2, 3, 4, 5):
    d = json.loads(open(os.path.join(ROOT, "profiles", f"r02_bench_cfg{c}.json")).read().strip().splitlines()[-1])
    print(f"| {names[c]} | {d['config']['L']:.3g} | {d['ms_per_step']:.3g} | {d['value']/1e9:.3g} | {d['path_roofline']['frac']:.3f} | "
          f"{d['roofline']['kernel']} ({d['roofline']['frac']:.2f}) | {d['e2e']['ms_per_step']:.3g} |")
d = json.loads(open(os.path.join(ROOT, "profiles", "r02_bench_cfg4.json")).read().strip().splitlines()[-1])
print(json.dumps({k: round(v, 3) for k, v in d["kernel_ms"].items()}))
print("cpu", d["cpu_baseline"]["value"] / 1e9, d["cpu_baseline"]["serial"]["value"] / 1e9, "e2e", d["e2e"])
print("roofline", d["roofline"], d["path_roofline"])
print("sharded", d.get("sharded_config_1gpu"))
