"""Warp-stall samples of a kernel in an ncu report, attributed to CUDA source lines.

ncu's SASS page (per-instruction samples) is mapped to source lines with the line table of the
same cubin (nvdisasm -gi; the binary that ran must be the in-tree libfikit.so).  Inlined code is
attributed to the innermost line and to the call site in the kernel's own file.
  python scripts/ncu_hot.py gpurun_out/x.ncu-rep k_prep [N]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
col = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"  # or "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address" and len(r) > 3][0]
h = rows[hi]
si = h.index(col)
samples = []
for r in rows[hi + 1:]:
    try:
        samples.append((int(r[0], 16), int(float(r[si].replace(",", ""))), r[1].strip()))
    except (ValueError, IndexError):
        pass
# one entry per instruction (the page can repeat rows per function instance)
seen = collections.OrderedDict()
for a, s, t in samples:
    if a not in seen:
        seen[a] = (s, t)
base = min(seen)
# line table of the kernel's function in the in-tree library
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2311_10359_b200", "libfikit.so")], cwd=tmp,
               capture_output=True)
where = {}
for cub in os.listdir(tmp):
    dis = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    cur_fn, inner, outer, fresh = None, None, None, True
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:  # a group of annotations: the first is the innermost line, the last the kernel's own
            tag = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            if fresh:
                inner = tag
                fresh = False
            outer = tag
            continue
        fresh = True
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m and cur_fn and kern in cur_fn:
            where[int(m.group(1), 16)] = (inner, outer)
tot = sum(s for s, _ in seen.values()) or 1
by_inner, by_outer = collections.Counter(), collections.Counter()
for a, (s, t) in seen.items():
    inner, outer = where.get(a - base, ("?", "?"))
    by_inner[inner] += s
    by_outer[outer] += s


def src_line(tag):
    f, _, l = tag.partition(":")
    for d in ("paper_2311_10359_b200/csrc", "include"):
        p = os.path.join(ROOT, d, f)
        if os.path.exists(p) and l.isdigit():
            return open(p).read().splitlines()[int(l) - 1].strip()[:90]
    return ""


print(f"{kern}: {tot} samples, {len(seen)} instructions")
print("-- innermost source line")
for tag, s in by_inner.most_common(n):
    print(f"{100 * s / tot:5.1f}%  {tag:22s} {src_line(tag)}")
print("-- call site in the kernel")
for tag, s in by_outer.most_common(n // 2):
    print(f"{100 * s / tot:5.1f}%  {tag:22s} {src_line(tag)}")
