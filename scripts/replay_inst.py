"""profiles/replay_inst.json: warp-instructions per scenario of the replay kernels (ncu
smsp__inst_executed.sum of one step's fikit_simulate_batch launches / the step's scenarios), the
count bench.py's replay_roofline multiplies by the live scenario rate.

  on the GPU box:  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum -k regex:k_simulate --csv \\
                     --log-file gpurun_out/replay_inst_<wl>.csv python bench.py --workload <wl> --steps 1 \\
                     --warmup 1 --no-e2e --no-cpu-baseline --no-configs2
  here:            python scripts/replay_inst.py <wl>=<scenarios> ...
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_p = os.path.join(ROOT, "profiles", "replay_inst.json")
out = json.load(open(out_p)) if os.path.exists(out_p) else {}
for spec in sys.argv[1:]:
    wl, S = spec.split("=")
    path = os.path.join(ROOT, "gpurun_out", f"replay_inst_{wl}.csv")
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = {}
    for r in rows[hi + 1:]:
        launches.setdefault(int(r[0]), {"kernel": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(launches)
    # the last step: the final fikit_simulate_batch call = its last two launches (reg + smem pass)
    last = [launches[i] for i in ids[-2:]]
    inst = sum(x["smsp__inst_executed.sum"] for x in last)
    out[wl] = {"warp_inst_per_scenario": inst / int(S), "kernels": [x["kernel"] for x in last],
               "ncu_ns": [x.get("gpu__time_duration.sum") for x in last],
               "source": f"ncu smsp__inst_executed.sum, {os.path.basename(path)} (last step's replay launches)"}
    print(wl, out[wl])
json.dump(out, open(out_p, "w"), indent=1)
