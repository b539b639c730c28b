"""Markdown table of the bench lines in a directory (bench_<config>.json written by tools/final_benches.sh)."""
import json, os, sys
d = sys.argv[1]
names = ["c0_2d_const", "c1_2d_rot", "c2_4d_stream", "c3_4d_lshape", "c4_6d_stream"]
print("| config | L | active DOF | DOF-applies/s | ms / step | steps/s | outer its / step | inner its / step | fp64 frac | HBM view | apply share | e2e (host trace) | DRAM B / DOF-apply | oracle (host cores) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for i, n in enumerate(names):
    p = os.path.join(d, f"bench_{n}.json")
    if not os.path.exists(p):
        continue
    b = json.load(open(p))
    r = b["roofline"]
    cpu = b.get("cpu_baseline", {}).get("value")
    print(f"| {n} (configs[{i}]) | {b['config']['L']} | {b['config']['dof_active']:,} | {b['value']:.3e} | {b['ms_per_step']:.1f} | "
          f"{b['time_steps_per_s']:.4g} | {b['outer_iters'] / b['steps']:.1f} | {b['inner_iters'] / b['steps']:.0f} | "
          f"{r['frac']:.4f} | {r['hbm_view']['frac']:.4f} | {r['share_of_step']:.2f} | {b['e2e']['value']:.3e} | "
          f"{r['traffic'] / r['dof_per_launch']:.1f} | {cpu:.3e} |" if cpu else "")
