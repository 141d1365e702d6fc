"""Summarise gpurun_out/ (ncu launch list + full captures + bench line) into profiles/<round>/.

  python scripts/summarize_profiles.py r01 <tag>
"""
import csv
import collections
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_requests_srcunit_tex_op_red.sum",
        "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = []
    for n, v in agg.items():
        lines.append(f"{n[:58]:58s} launches={len(v):4d} avg_us={sum(v) / len(v) / 1e3:9.1f} share={sum(v) / tot * 100:5.1f}%")
    return lines


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = dict(zip(h, v))
    U = dict(zip(h, u))
    st = []
    for k, x in d.items():
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(x.replace(",", "")), k.replace("smsp__average_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    return [(k, d.get(k), U.get(k)) for k in KEYS], st[:6]


def main():
    rnd, tag = sys.argv[1], sys.argv[2]
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    lines = [f"# {tag}: ncu summaries (from gpurun_out/, scripts/summarize_profiles.py)", ""]
    bj = os.path.join(OUT, "bench.json")
    if os.path.exists(bj) and os.path.getsize(bj):
        b = json.load(open(bj))
        lines += ["## bench.py line (N=1)", "", "```", json.dumps(b, indent=1), "```", ""]
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        lines += ["## launch list: `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 3 "
                  "--warmup 1 --no-e2e --no-cpu-baseline` (cold-cache, serialised: compare SHARES)", "", "```"]
        lines += launches(lc) + ["```", ""]
    for f in sorted(os.listdir(OUT)):
        if f.startswith("prof_") and f.endswith(".ncu-rep"):
            kv, st = raw(os.path.join(OUT, f))
            lines += [f"## `ncu --set full` capture {f} (1 launch)", "", "| metric | value | unit |", "|---|---|---|"]
            lines += [f"| {k} | {v} | {u} |" for k, v, u in kv]
            lines += ["", "top stall reasons (cycles per issued instruction): " +
                      ", ".join(f"{n} {x:.2f}" for x, n in st), ""]
    path = os.path.join(dst, f"{tag}.md")
    open(path, "w").write("\n".join(lines) + "\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
