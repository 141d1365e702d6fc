"""Write tests/golden/toy_oracle.json: configs[0] (toy) through the oracle.

Calls only oracle/ and fikit_synth/ (never the CUDA path).  Re-run after a
justified oracle change:  python tests/golden/make_toy.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import fikit_synth as F  # noqa: E402
import oracle  # noqa: E402


def main():
    cfg = F.toy()
    out = {"source": "make_toy.py: fikit_synth.toy(seed=1) through oracle/ (measure, resolve, simulate)"}
    for fb in (1, 0):
        cfg.replay.feedback = fb
        r = oracle.pipeline(cfg)
        t = r["table"].head()
        out["table"] = {k: v.tolist() for k, v in t.items()}
        out["status"] = r["status"]
        res = r["results"][0]
        out[f"feedback{fb}"] = {"result": {k: int(res[k]) for k in res.dtype.names},
                                "fill_gap": r["fill_gap"].tolist(), "lp_start": r["lp_start"].tolist()}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "toy_oracle.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
