import sys, numpy as np
sys.path.insert(0, '.')
import fikit_synth as F, oracle
import paper_2311_10359_b200 as fk
from paper_2311_10359_b200.pipeline import Pipeline
cfg = F.resnet_trace(n_runs=int(sys.argv[1]) if len(sys.argv) > 1 else 10000)
tr = cfg.trace
for rep in range(3):
    p = Pipeline(tr.records, tr.names, tr.sigs, capacity=4096)
    fk.measure(p.recs, p.n, p.names, p.sigs, p.table, p.ws)
    st = fk.get_status(p.ws)
    import torch
    torch.cuda.synchronize()
    n = st['n_rows_needed']
    kid = p.table.kernel_id.cpu().numpy().view(np.uint64)[:n]
    task = p.table.task_id.cpu().numpy()[:n]
    ref, _ = oracle.identify(tr.records, tr.names, tr.sigs)
    refset = set(zip(tr.records['task_id'].tolist(), ref.tolist()))
    got = list(zip(task.tolist(), kid.tolist()))
    dup = len(got) - len(set(got))
    garbage = sum(1 for g in got if g not in refset)
    print(f"rep {rep}: n_rows_needed={n} distinct_ref={len(refset)} dup={dup} garbage={garbage} status={st}")
    # hot dictionary size
    ws = p.ws.t.cpu().numpy()
