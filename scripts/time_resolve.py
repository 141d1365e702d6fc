"""Time fikit_resolve (HP + LP launches of the Zipf replay leg in one call) on one GPU, and print
a checksum of its outputs (to compare library variants: FIKIT_DIAG_LIB=<lib> python ...).

  python scripts/time_resolve.py [--records N]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import fikit_synth as F  # noqa: E402
import paper_2311_10359_b200 as fk  # noqa: E402
from paper_2311_10359_b200.pipeline import Pipeline  # noqa: E402

N = int(sys.argv[sys.argv.index("--records") + 1]) if "--records" in sys.argv else 12_500_000
cfg = F.zipf_trace(n_runs=max(1, N // 256), threads=16)
rp = F.zipf_replay(cfg)
p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=8192, replay=rp)
p.step()
p.check("step")
r = p.replay
call = lambda: fk.resolve(r["recs_both"], r["nh"] + r["nl"], p.names, p.sigs, p.table, r["row_both"], r["dur_both"],
                          r["gap_both"], p.ws, reuse_hashes=True)
for _ in range(3):
    call()
torch.cuda.synchronize()
sums = [int(t.cpu().numpy().view(np.uint64 if t.element_size() == 8 else np.uint32).astype(np.uint64).sum())
        for t in (r["row_both"], r["dur_both"], r["gap_both"])]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(7):
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 20)
print(f"{os.environ.get('FIKIT_DIAG_LIB', 'in-tree')}: resolve of {r['nh'] + r['nl']:,} launches {best * 1e3:.1f} us "
      f"(rows of {p.table.n_rows()}); checksums {sums}")
