"""A/B timing of fikit_simulate_batch across replay.cu variants in ONE process on one GPU.

  python scripts/ab_replay.py build           (here, CPU: abtest_replay/<name>/libfikit.so from the working tree)
  python scripts/ab_replay.py run [--records N] [--scenarios S]   (on the GPU)

The table and resolved inputs come from the in-tree library (zipf trace + zipf replay, as in
bench.py); every variant replays the same device inputs and its results are compared bytewise
with the in-tree library's.
"""
import ctypes as C
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AB = os.path.join(ROOT, "abtest_replay")
CS = "paper_2311_10359_b200/csrc/"
sys.path.insert(0, ROOT)


def sub(txt, old, new):
    assert old in txt, old[:80]
    return txt.replace(old, new)


def reg_cfg(warps, minb):
    def f(r, h):
        h = sub(h, "constexpr int kRegThreads = 512;", f"constexpr int kRegThreads = {warps * 32};")
        r = sub(r, "__launch_bounds__(kRegWarps * 32, 2)", f"__launch_bounds__(kRegWarps * 32, {minb})")
        return r, h
    return f


VARIANTS = {
    "base": [],  # 16 warps, 2 blocks per SM (64 registers)
    "w8b2": [reg_cfg(8, 2)],  # 16 warps per SM, up to 128 registers
    "w4b6": [reg_cfg(4, 6)],
    "w16b1": [reg_cfg(16, 1)],
    "w4b5": [reg_cfg(4, 5)],  # 20 warps per SM, up to 102 registers
    "w4b7": [reg_cfg(4, 7)],  # 28 warps per SM, up to 72 registers
    "w4b8": [reg_cfg(4, 8)],  # 32 warps per SM, up to 64 registers
    "w8b4": [reg_cfg(8, 4)],
    "w16b2": [reg_cfg(16, 2)],
    # register pool: a dequeue clears only pq (Rc capped at 0xFFFFFFFE, so a cleared pq never fits)
    "deq": [lambda r, h: (sub(sub(r,
        "const uint32_t Rc = R >= (1u << 22) ? 0xFFFFFFFFu : (R << 6) | 63u;",
        "const uint32_t Rc = R >= (1u << 22) ? 0xFFFFFFFEu : (R << 6) | 63u;"),
        "if (k < 32u) key0 = pq0 = 0xFFFFFFFFu; else key1 = pq1 = 0xFFFFFFFFu;",
        "if (k < 32u) pq0 = 0xFFFFFFFFu; else pq1 = 0xFFFFFFFFu;"), h)],
    # register pool: no "nothing fits" checks after the pick (the caller's R >= qmin guarantees a fit)
    "nofitchk": [lambda r, h: (sub(sub(r,
        "    if (best == 0xFFFFFFFFu) return -1;\n    const uint32_t k = best & 63u;",
        "    const uint32_t k = best & 63u;"),
        "      const int k = P.pick32(R, lane, qk);  // Alg. 2\n      if (k < 0) break;",
        "      const int k = P.pick32(R, lane, qk);  // Alg. 2 (R >= qmin: one fits)"), h)],
    # the POOL models' HP chunk walk without the lazy (REDUX-total) path: the prefix scan every chunk
    "eager": [lambda r, h: (sub(r, "template <bool kLazyScan = true, class GateMin, class Fill>",
                                "template <bool kLazyScan = false, class GateMin, class Fill>"), h)],
}


def build(names):
    os.makedirs(AB, exist_ok=True)
    for name in names:
        d = os.path.join(AB, name)
        src = os.path.join(d, "src")
        os.makedirs(os.path.join(src, CS), exist_ok=True)
        os.makedirs(os.path.join(src, "include"), exist_ok=True)
        for f in ("measure.cu", "finalize.cu", "capi.cu"):
            shutil.copy(os.path.join(ROOT, CS, f), os.path.join(src, CS, f))
        shutil.copy(os.path.join(ROOT, "include/fikit.h"), os.path.join(src, "include/fikit.h"))
        r = open(os.path.join(ROOT, CS, "replay.cu")).read()
        h = open(os.path.join(ROOT, CS, "fikit_internal.cuh")).read()
        for t in VARIANTS[name]:
            r, h = t(r, h)
        open(os.path.join(src, CS, "replay.cu"), "w").write(r)
        open(os.path.join(src, CS, "fikit_internal.cuh"), "w").write(h)
        objs = []
        for f in ("measure.cu", "finalize.cu", "replay.cu", "capi.cu"):
            o = os.path.join(d, f + ".o")
            res = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                                  "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-c",
                                  os.path.join(src, CS, f), "-o", o], capture_output=True, text=True)
            if res.returncode:
                print(name, "FAILED", res.stderr[-2000:])
                raise SystemExit(1)
            if f == "replay.cu":
                lines = res.stderr.splitlines()
                info = []
                for k, ln in enumerate(lines):
                    if "Compiling" in ln and "k_simulate" in ln:
                        info += [x.strip() for x in lines[k:k + 4] if "registers" in x or "spill" in x]
                print(name, info)
            objs.append(o)
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-o", os.path.join(d, "libfikit.so"), *objs])


def run(records, S):
    import torch

    import fikit_synth as F
    import paper_2311_10359_b200 as fk
    from paper_2311_10359_b200.pipeline import Pipeline

    cfg = F.zipf_trace(n_runs=max(1, records // 256))
    rp = F.zipf_replay(cfg, S=S)
    p = Pipeline(cfg.trace.records, cfg.trace.names, cfg.trace.sigs, capacity=8192, replay=rp)
    p.step()
    torch.cuda.synchronize()
    r = p.replay
    ref = r["out"].clone()
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for name in sorted(os.listdir(AB)):
        path = os.path.join(AB, name, "libfikit.so")
        if not os.path.exists(path):
            continue
        L = C.CDLL(path)
        L.fikit_simulate_batch.argtypes = [C.POINTER(fk.TableC)] + [C.c_void_p] * 7 + [C.c_uint32, fk.FillParamsC] + \
            [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p]
        prm = fk.FillParamsC(r["threshold_ns"], r["feedback"], 0)
        out = torch.zeros_like(ref)
        call = lambda: L.fikit_simulate_batch(C.byref(p.table.c), ptr(r["hp_row"]), ptr(r["hp_dur"]),
                                              ptr(r["hp_gap"]), ptr(r["lp_row"]), ptr(r["lp_dur"]),
                                              ptr(r["lp_level"]), ptr(r["sc"]), r["S"], prm, ptr(out), None, None,
                                              None, p.ws.ptr(), p.ws.nbytes, stream)
        for _ in range(3):
            rc = call()
        torch.cuda.synchronize()
        same = bool(torch.equal(out, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        for _ in range(5):
            e0.record()
            for _ in range(10):
                call()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 10)
        print(name, json.dumps({"ms": min(times), "rc": rc, "same_as_intree": same}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:] or list(VARIANTS))
    else:
        rec = int(sys.argv[sys.argv.index("--records") + 1]) if "--records" in sys.argv else 4_000_000
        S = int(sys.argv[sys.argv.index("--scenarios") + 1]) if "--scenarios" in sys.argv else 100_000
        run(rec, S)
