"""A pipeline step captured into a CUDA graph (as bench.py times it) gives the oracle's results on
every replay: measure + finalize + resolve + replay through the C-ABI under stream capture, the
timed variant's events recorded as external nodes (include/fikit.h), replayed several times on
the same inputs.  Expected values come from the oracle (oracle/) on the same inputs."""
import numpy as np
import pytest

import fikit_synth as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fk():
    from conftest import cuda_ok

    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2311_10359_b200 as fk
    from paper_2311_10359_b200 import _build

    _build.build()
    return fk


@pytest.mark.parametrize("kind", ["toy", "bert_vgg"])
def test_graph_step_matches_oracle(fk, orc, kind):
    import torch

    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.toy() if kind == "toy" else F.bert_vgg(S=3000)
    cap = 64 if kind == "toy" else 1024
    ref = orc.pipeline(cfg, capacity=cap)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=cap, replay=cfg.replay)
    p.step()  # (direct launches once: the workspace then holds the string hashes resolve reuses)
    p.check("direct step")
    ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
    for e in ev:
        e.record()
    n0 = fk.launch_count()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fk.measure(p.recs, p.n, p.names, p.sigs, p.table, p.ws, events=ev)
        fk.table_finalize(p.table, p.ws)
        p.run_replay()
    assert fk.launch_count() > n0  # the calls launched (into the graph)
    for rep in range(3):
        p.table.block.zero_()  # (the replay must rebuild the table from scratch)
        p.replay["out"].zero_()
        g.replay()
        torch.cuda.synchronize()
        assert ev[0].elapsed_time(ev[1]) > 0  # the external event nodes time k_measure on replay
        st = p.check(f"graph replay {rep}")
        got = p.table.to_numpy()
        for k, v in ref["table"].head().items():
            assert np.array_equal(got[k], v), f"{kind} replay {rep}: table field {k}"
        assert p.results().tobytes() == ref["results"].tobytes(), f"{kind} replay {rep}: results"
        assert st["code"] == 0
