"""Decode / small-M probe (GPU box; perf probing): BASELINE config 1 (6:8
INT8 4096x4096, M=128) and config 4 (Llama-3.1-8B 6:8 BF16, M=1/16/64).
Each op is its own CUDA graph, timed after a 512 MiB L2-flush write (CUDA
events, median of reps); prints the tile config, µs and weight-stream GB/s
for lift, sparse GEMM, lift+sparse as one graph, and the dense GEMM (+ its
activation quantization for INT8)."""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

LLAMA8 = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
FLUSH = None


def graph(fns):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    return g


def t_us(fns, reps):
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    g = graph(fns)
    evs = []
    for _ in range(reps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in evs) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--cfg", default="1,4")
    ap.add_argument("--ms", default="1,16,64")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    if "1" in a.cfg.split(","):
        n = k = 4096
        m = 128
        w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
        pw = slsp.pack_compress(w, 6, 8)
        x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        pay, st = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp)
        q, qs = slsp.quantize_rows(x)
        ys = torch.empty((n, m), dtype=torch.int32, device="cuda")
        lift = lambda: slsp.fused_quant_slide(x, 6, 8, kp=pw.kp, check=False, payload=pay, scales=st)
        gemm = lambda: slsp.sparse_gemm(pw, pay, out=ys)
        quant = lambda: slsp.quantize_rows(x, check=False, out=q, scales=qs)
        dgemm = lambda: slsp.dense_gemm(w, q.view(torch.int8), out=ys)
        sb = n * pw.kp // 2 + n * pw.kp // 8 + m * pw.kp + n * m * 4
        db = n * k + m * k + n * m * 4
        r = {"case": "cfg1 int8 4096x4096 M=128", "config": slsp.sparse_gemm_config(pw, m),
             "lift_us": t_us([lift], a.reps), "sparse_us": t_us([gemm], a.reps), "step_us": t_us([lift, gemm], a.reps),
             "dense_us": t_us([dgemm], a.reps), "dense_step_us": t_us([quant, dgemm], a.reps)}
        r["sparse_gbs"] = sb / r["sparse_us"] / 1e3
        r["dense_gbs"] = db / r["dense_us"] / 1e3
        rows.append(r)
    if "4" in a.cfg.split(","):
        for name, n, k in LLAMA8:
            w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
            pw = slsp.pack_compress(w, 6, 8)
            for m in [int(v) for v in a.ms.split(",")]:
                x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
                lifted = slsp.lift_rows(x, 6, 8, kp=pw.kp)
                ys = slsp.sparse_gemm(pw, lifted)
                yd = slsp.dense_gemm(w, x)
                lift = lambda: torch.ops.aten.copy_(lifted, slsp.lift_rows(x, 6, 8, kp=pw.kp)) if False else \
                    slsp._native.lib().slsp_lift_rows(slsp.DT_BF16, slsp._native._ptr(x), m, k, 6, 8, pw.kp,
                                                      slsp._native._ptr(lifted), slsp._native._stream(x.device))
                gemm = lambda: slsp.sparse_gemm(pw, lifted, out=ys)
                dgemm = lambda: slsp.dense_gemm(w, x, out=yd)
                sb = n * pw.kp // 2 * 2 + n * pw.kp // 8 + m * pw.kp * 2 + n * m * 4
                db = n * k * 2 + m * k * 2 + n * m * 4
                r = {"case": f"cfg4 bf16 {name} {n}x{k} M={m}", "config": slsp.sparse_gemm_config(pw, m),
                     "lift_us": t_us([lift], a.reps), "sparse_us": t_us([gemm], a.reps),
                     "step_us": t_us([lift, gemm], a.reps), "dense_us": t_us([dgemm], a.reps)}
                r["dense_step_us"] = r["dense_us"]
                r["sparse_gbs"] = sb / r["sparse_us"] / 1e3
                r["dense_gbs"] = db / r["dense_us"] / 1e3
                rows.append(r)
    for r in rows:
        r["step_speedup"] = r["dense_step_us"] / r["step_us"]
        r["gemm_speedup"] = r["dense_us"] / r["sparse_us"]
        c = r.pop("config")
        r["cfg"] = f"bn{c['tokens_per_tile']} ms{c['subtiles']} ks{c['ksplit']} st{c['stages']} cl{c['clusters']}"
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)


if __name__ == "__main__":
    main()
