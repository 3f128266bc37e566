"""In-SM lifting (sparse_gemm_x: unlifted quantized X, the lifted window
built in shared memory) vs the lifted-operand sparse GEMM and the dense GEMM
at moderate M (config 3's regime, where one-subtile tiles are bound by the
bytes each SM ingests). CUDA-event medians, L2 flushed before each launch
(perf probing)."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

QWEN7 = {"qkv": (4608, 3584), "o": (3584, 3584), "gate_up": (37888, 3584), "down": (3584, 18944)}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


g = torch.Generator(device="cuda").manual_seed(0)
ms = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512,1024,2048,8192").split(",")]
for name, (n, k) in QWEN7.items():
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    go = pw.gemm_order()
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01
    for m in ms:
        x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        pay, st = slsp.fused_quant_slide(x, 6, 8)
        qx, qs = slsp.quantize_rows(x, kpad=go.kx)
        q, q_s = slsp.quantize_rows(x)
        out = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
        y1 = slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=st, out_mode=slsp.OUT_BF16_NM)
        y2 = slsp.sparse_gemm_x(go, qx, s_ch=s_ch, s_tok=qs, out_mode=slsp.OUT_BF16_NM)
        same = bool(torch.equal(y1.view(torch.int16), y2.view(torch.int16)))
        t_s = timed(lambda: slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=st, out_mode=slsp.OUT_BF16_NM, out=out))
        t_x = timed(lambda: slsp.sparse_gemm_x(go, qx, s_ch=s_ch, s_tok=qs, out_mode=slsp.OUT_BF16_NM, out=out))
        t_d = timed(lambda: slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=q_s, out_mode=slsp.OUT_BF16_NM,
                                            out=out))
        t_l = timed(lambda: slsp.fused_quant_slide(x, 6, 8, check=False, payload=pay, scales=st))
        t_q = timed(lambda: slsp.quantize_rows(x, kpad=go.kx, check=False, out=qx, scales=qs))
        print(json.dumps({"layer": name, "m": m, "sparse_us": round(t_s, 2), "insm_us": round(t_x, 2),
                          "dense_us": round(t_d, 2), "lift_us": round(t_l, 2), "quant_us": round(t_q, 2),
                          "gemm_speedup": round(t_d / t_s, 3), "insm_speedup": round(t_d / t_x, 3),
                          "identical": same}), flush=True)
