"""Decode / small-M in steady state (GPU box; perf probing): each case runs
as one CUDA graph of R back-to-back layer calls over C distinct weight
copies (C * weight bytes > 2x L2, so every call streams its weights from
HBM, as in a decode step), timed with CUDA events; per-call µs = total / R.
Sparse step = lift (or quant) + GEMM per call; dense step = GEMM (BF16) or
quantize_rows + GEMM (INT8). Knob configs (SLSP_GEMM_* env) are swept in
one process: --knobs 'SPLITCOST=32;SPLITCOST=4;KSPLIT=1'."""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

LLAMA8 = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
L2 = 126 << 20


def run_graph(fns, reps=5):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def apply(kv):
    for k in list(os.environ):
        if k.startswith("SLSP_GEMM_") or k.startswith("SLSP_DGEMM_") or k == "SLSP_PDL":
            del os.environ[k]
    for k, v in kv.items():
        os.environ[("SLSP_" if k == "PDL" else "SLSP_GEMM_") + k] = v
    slsp.reload_knobs()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg1,qkv,o,gate_up,down")
    ap.add_argument("--ms", default="1,16,64")
    ap.add_argument("--calls", type=int, default=40)
    ap.add_argument("--knobs", default="")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    knobs = [dict(x.split("=") for x in part.split() if "=" in x) for part in a.knobs.split(";")] if a.knobs else [{}]
    for case in a.cases.split(","):
        if case == "cfg1":
            n, k, ms, bf16 = 4096, 4096, [128], False
        else:
            (n, k), ms, bf16 = LLAMA8[case], [int(v) for v in a.ms.split(",")], True
        wbytes = n * k * (2 if bf16 else 1)
        copies = max(2, -(-2 * L2 // wbytes))
        ws, pws = [], []
        for _ in range(copies):
            if bf16:
                w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
            else:
                w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g),
                                         6, 8)
            ws.append(w)
            pws.append(slsp.pack_compress(w, 6, 8))
        kp = pws[0].kp
        for m in ms:
            x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            for kv in knobs:
                apply(kv)
                cfg = slsp.sparse_gemm_config(pws[0], m)
                if bf16:
                    lifted = slsp.lift_rows(x, 6, 8, kp=kp)
                    ys = torch.empty((n, m), dtype=torch.float32, device="cuda")
                    lib, N = slsp.lib(), slsp._native
                    lift = lambda: lib.slsp_lift_rows(slsp.DT_BF16, N._ptr(x), m, k, 6, 8, kp, N._ptr(lifted),
                                                      N._stream(x.device))
                    sp = [f for i in range(a.calls) for f in (lift, (lambda j: lambda: slsp.sparse_gemm(
                        pws[j], lifted, out=ys))(i % copies))]
                    sp_g = [(lambda j: lambda: slsp.sparse_gemm(pws[j], lifted, out=ys))(i % copies)
                            for i in range(a.calls)]
                    de = [(lambda j: lambda: slsp.dense_gemm(ws[j], x, out=ys))(i % copies) for i in range(a.calls)]
                    gl = [(lambda j: lambda: slsp.sparse_gemm_lift(pws[j], x, out=ys))(i % copies)
                          for i in range(a.calls)]
                else:
                    gl = None
                    pay, st = slsp.fused_quant_slide(x, 6, 8, kp=kp)
                    q, qs = slsp.quantize_rows(x)
                    ys = torch.empty((n, m), dtype=torch.int32, device="cuda")
                    lift = lambda: slsp.fused_quant_slide(x, 6, 8, kp=kp, check=False, payload=pay, scales=st)
                    quant = lambda: slsp.quantize_rows(x, check=False, out=q, scales=qs)
                    sp = [f for i in range(a.calls) for f in (lift, (lambda j: lambda: slsp.sparse_gemm(
                        pws[j], pay, out=ys))(i % copies))]
                    sp_g = [(lambda j: lambda: slsp.sparse_gemm(pws[j], pay, out=ys))(i % copies)
                            for i in range(a.calls)]
                    de = [f for i in range(a.calls) for f in (quant, (lambda j: lambda: slsp.dense_gemm(
                        ws[j], q.view(torch.int8), out=ys))(i % copies))]
                t_sp = run_graph(sp) / a.calls
                t_g = run_graph(sp_g) / a.calls
                t_de = run_graph(de) / a.calls
                t_gl = run_graph(gl) / a.calls if gl else None
                sb = n * kp // 2 * (2 if bf16 else 1) + n * kp // 8
                db = n * k * (2 if bf16 else 1)
                print(json.dumps({"case": f"{case} {n}x{k} M={m}", "knobs": kv, "sparse_step_us": round(t_sp, 2),
                                  "sparse_gemm_us": round(t_g, 2), "dense_step_us": round(t_de, 2),
                                  "step_speedup": round(t_de / t_sp, 3),
                                  "glift_step_us": round(t_gl, 2) if t_gl else None,
                                  "glift_speedup": round(t_de / t_gl, 3) if t_gl else None,
                                  "gemm_weight_gbs": round(sb / t_g / 1e3, 1), "dense_weight_gbs": round(db / t_de / 1e3, 1),
                                  "cfg": f"bn{cfg['tokens_per_tile']} ks{cfg['ksplit']} ksc{cfg['cluster_ksplit']} cl{cfg['clusters']}"}),
                      flush=True)


if __name__ == "__main__":
    main()
