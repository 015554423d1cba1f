"""One-line summary of a bench.py JSON line: python tools/bench_summary.py gpurun_out/bench.log"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: (round(d[k], 2) if isinstance(d[k], float) else d[k]) for k in
       ["value", "ms_per_step", "filter_kernel_gflops", "gpu_launches"]})
print("roofline frac", round(d["roofline"]["frac"], 3), "e2e", d.get("e2e") and round(d["e2e"]["value"], 1),
      "cpu", d.get("cpu_baseline") and round(d["cpu_baseline"]["value"], 1), "clocks", d.get("clocks"))
tot = {}
for p in d["per_problem"]:
    for k, v in p["dev_ms"].items():
        tot[k] = tot.get(k, 0) + v
    for k in ("t_reduce_ms", "t_back_ms", "t_solve_ms"):
        tot[k] = tot.get(k, 0) + p[k]
print({k: round(v, 1) for k, v in tot.items()}, "loops", [p["loops"] for p in d["per_problem"]])
