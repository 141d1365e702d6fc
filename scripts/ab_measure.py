"""A/B timing of fikit_measure across library variants in ONE process on one GPU.

  python scripts/ab_measure.py build <name>=<git-rev> ...   (here, CPU: builds build/ab/<name>/libfikit.so)
  python scripts/ab_measure.py run [--records N]             (on the GPU: times every built variant)
"""
import ctypes as C
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
AB = os.path.join(ROOT, "ab_out")  # (git-ignored, but shipped to the GPU box by gpurun)
sys.path.insert(0, ROOT)


def build(specs):
    for spec in specs:
        # name=rev[+DEFINE[+DEFINE...]]; rev "." = the working tree
        name, rev = spec.split("=", 1)
        rev, *defs = rev.split("+")
        d = os.path.join(AB, name)
        src = os.path.join(d, "src")
        os.makedirs(os.path.join(src, "paper_2311_10359_b200", "csrc"), exist_ok=True)
        os.makedirs(os.path.join(src, "include"), exist_ok=True)
        files = ["paper_2311_10359_b200/csrc/" + f for f in
                 ("measure.cu", "finalize.cu", "replay.cu", "capi.cu", "fikit_internal.cuh")] + ["include/fikit.h"]
        for f in files:
            data = (open(os.path.join(ROOT, f), "rb").read() if rev == "." else
                    subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:{f}"]))
            open(os.path.join(src, f), "wb").write(data)
        objs = []
        for f in ("measure.cu", "finalize.cu", "replay.cu", "capi.cu"):
            o = os.path.join(d, f + ".o")
            subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                                   "-std=c++17", "-Xcompiler", "-fPIC", *[f"-D{x}" for x in defs], "-c",
                                   os.path.join(src, "paper_2311_10359_b200", "csrc", f), "-o", o])
            objs.append(o)
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-o", os.path.join(d, "libfikit.so"), *objs])
        print("built", name, rev)


def run(records, workload="zipf"):
    import numpy as np
    import torch

    import fikit_synth as F
    import paper_2311_10359_b200 as fk

    if workload == "resnet":
        cfg = F.resnet_trace(n_runs=max(1, records // 300))
    else:
        cfg = F.zipf_trace(n_runs=max(1, records // 256))
    tr = cfg.trace
    n = tr.records.shape[0]
    recs = fk.records_to_device(tr.records)
    names, sigs = fk.strtab_to_device(tr.names), fk.strtab_to_device(tr.sigs)
    out = {}
    variants = []
    for name in sorted(os.listdir(AB)):
        path = os.path.join(AB, name, "libfikit.so")
        if not os.path.exists(path):
            continue
        L = C.CDLL(path)
        L.fikit_ws_bytes.restype = C.c_size_t
        L.fikit_ws_bytes.argtypes = [C.c_uint32] * 3 + [C.c_uint64]
        L.fikit_table_bytes.restype = C.c_size_t
        L.fikit_table_bytes.argtypes = [C.c_uint32]
        L.fikit_table_carve.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(fk.TableC)]
        L.fikit_measure_timed.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, fk.StrTabC, fk.StrTabC,
                                          C.POINTER(fk.TableC), C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.fikit_get_status.argtypes = [C.c_void_p, C.POINTER(fk.StatusC), C.c_void_p]
        L.fikit_table_finalize.argtypes = [C.POINTER(fk.TableC), C.c_void_p, C.c_uint64, C.c_void_p, C.c_size_t,
                                           C.c_void_p]
        cap = 8192
        wsb = L.fikit_ws_bytes(cap, names.count, sigs.count, n)
        ws = torch.empty(wsb + 256, dtype=torch.uint8, device="cuda")
        wsp = ws.data_ptr() + (-ws.data_ptr()) % 256
        tb = torch.zeros(L.fikit_table_bytes(cap) + 256, dtype=torch.uint8, device="cuda")
        t = fk.TableC()
        L.fikit_table_carve(C.c_void_p(tb.data_ptr() + (-tb.data_ptr()) % 256), cap, C.byref(t))
        variants.append((name, L, ws, wsp, wsb, tb, t))
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record()
    k1.record()

    def call(v, ev=(None, None)):
        name, L, ws, wsp, wsb, tb, t = v
        return L.fikit_measure_timed(C.c_void_p(recs.data_ptr()), n, None, names.c(), sigs.c(), C.byref(t), None,
                                     C.c_void_p(wsp), wsb, stream, ev[0], ev[1])

    for v in variants:
        for _ in range(3):
            call(v)
        torch.cuda.synchronize()
        st = fk.StatusC()
        v[1].fikit_get_status(C.c_void_p(v[3]), C.byref(st), stream)
        out[v[0]] = {"ms": [], "kernel_ms": [], "status": st.code, "rows": st.n_rows_needed}
        # the finalized table must be identical across variants (bytes of the whole table block)
        v[1].fikit_table_finalize(C.byref(v[6]), None, 0, C.c_void_p(v[3]), v[4], stream)
        torch.cuda.synchronize()
        blk = v[5].cpu().numpy()
        out[v[0]]["table_equal_first"] = bool(np.array_equal(blk, variants[0][5].cpu().numpy()))
    if os.environ.get("AB_ONCE"):  # for an ncu launch list: 3 calls each only
        return out
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(7):  # variants interleaved: clock / thermal drift hits all alike
        for v in variants:
            e0.record()
            kt = 0.0
            for _ in range(10):
                call(v, (C.c_void_p(k0.cuda_event), C.c_void_p(k1.cuda_event)))
            e1.record()
            torch.cuda.synchronize()
            out[v[0]]["ms"].append(e0.elapsed_time(e1) / 10)
            out[v[0]]["kernel_ms"].append(k0.elapsed_time(k1))  # (the last call's k_measure)
    # fikit_table_finalize alone (re-runnable: it reads the workspace's measured rows), interleaved
    for v in variants:
        call(v)
        out[v[0]]["fin_ms"] = []
    for rep in range(7):
        for v in variants:
            e0.record()
            for _ in range(20):
                v[1].fikit_table_finalize(C.byref(v[6]), None, 0, C.c_void_p(v[3]), v[4], stream)
            e1.record()
            torch.cuda.synchronize()
            out[v[0]]["fin_ms"].append(e0.elapsed_time(e1) / 20)
    for name, r in out.items():
        r["fin_ms"] = min(r["fin_ms"])
        r["ms"], r["kernel_ms"] = min(r["ms"]), float(np.median(r["kernel_ms"]))
        r["GBps_call"] = 48 * n / r["ms"] / 1e6
        r["GBps_kernel"] = 48 * n / r["kernel_ms"] / 1e6
        print(name, json.dumps(r), flush=True)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        rec = int(sys.argv[sys.argv.index("--records") + 1]) if "--records" in sys.argv else 100_000_000
        wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "zipf"
        run(rec, wl)
