"""§8f #3 chain timing (GPU box; perf probing): Qwen2.5-14B o_proj -> gate_up at
M tokens, INT8 6:8, token-major BF16 between the layers.

  unfused: sparse_gemm(o) -> fused_quant_slide(y1) -> sparse_gemm(gate_up)
  fused:   sparse_gemm(o, tok_amax) -> fused_quant_slide(y1, absmax) -> sparse_gemm(gate_up)

Each variant is one CUDA graph, timed after a 512 MiB L2-flush write (CUDA
events, median of reps); the lift alone is also timed in both forms with y1
L2-cold (flushed) and L2-warm (right after the GEMM that wrote it).
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402


def graph(fns):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for f in fns:
            f()
    return g


def timed(g, reps, flush, pre=None):
    evs = []
    for _ in range(reps):
        flush.zero_()
        if pre is not None:
            pre.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    m = a.m
    gen = torch.Generator(device="cuda").manual_seed(0)
    (n1, k1), (n2, k2) = (5120, 5120), (27648, 5120)

    def lay(n, k):
        w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=gen), 6, 8)
        return slsp.pack_compress(w, 6, 8), torch.rand(n, device="cuda", generator=gen) * 0.01 + 0.001

    p1, s1 = lay(n1, k1)
    p2, s2 = lay(n2, k2)
    x = (torch.rand(m, k1, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)
    pay1, t1 = slsp.fused_quant_slide(x, 6, 8, kp=p1.kp)
    y1 = torch.empty((m, n1), dtype=torch.bfloat16, device="cuda")
    y2 = torch.empty((n2, m), dtype=torch.bfloat16, device="cuda")
    amax = torch.empty(m, device="cuda")
    pay2 = torch.empty((m, p2.kp // 4), dtype=torch.int32, device="cuda")
    t2 = torch.empty(m, device="cuda")
    om = slsp.OUT_BF16_MN
    g1 = lambda: slsp.sparse_gemm(p1, pay1, s_ch=s1, s_tok=t1, out_mode=om, out=y1)
    g1a = lambda: slsp.sparse_gemm(p1, pay1, s_ch=s1, s_tok=t1, out_mode=om, out=y1, tok_amax=amax)
    lift = lambda: slsp.fused_quant_slide(y1, 6, 8, kp=p2.kp, check=False, payload=pay2, scales=t2)
    lifts = lambda: slsp.fused_quant_slide(y1, 6, 8, kp=p2.kp, check=False, payload=pay2, scales=t2, absmax=amax)
    g2 = lambda: slsp.sparse_gemm(p2, pay2, s_ch=s2, s_tok=t2, out_mode=slsp.OUT_BF16_NM, out=y2)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    G = {"unfused": graph([g1, lift, g2]), "fused": graph([g1a, lifts, g2]),
         "gemm1": graph([g1]), "gemm1_amax": graph([g1a]), "lift": graph([lift]), "lift_scaled": graph([lifts]),
         "gemm2": graph([g2])}
    res = {"m": m, "layers": "qwen2.5-14b o_proj 5120x5120 -> gate_up 27648x5120, 6:8 int8"}
    for _ in range(2):
        for name, g in G.items():
            res[name + "_ms"] = round(timed(g, a.reps, flush), 4)
        res["lift_warm_ms"] = round(timed(G["lift"], a.reps, flush, pre=G["gemm1"]), 4)
        res["lift_scaled_warm_ms"] = round(timed(G["lift_scaled"], a.reps, flush, pre=G["gemm1_amax"]), 4)
    import os
    os.environ["SLSP_GEMM_DEBUG"] = "256"
    slsp.reload_knobs()
    res["gemm1_amax_noatomic_ms"] = round(timed(graph([g1a]), a.reps, flush), 4)
    os.environ.pop("SLSP_GEMM_DEBUG")
    slsp.reload_knobs()
    ok = bool(torch.equal(pay2, slsp.fused_quant_slide(y1, 6, 8, kp=p2.kp)[0]))
    res["payload_identical"] = ok
    res["lift_bytes"] = m * (k2 * 2 + p2.kp + 4)
    res["lift_scaled_gbs"] = round(res["lift_bytes"] / res["lift_scaled_ms"] / 1e6, 1)
    res["lift_gbs"] = round(res["lift_bytes"] / res["lift_ms"] / 1e6, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
