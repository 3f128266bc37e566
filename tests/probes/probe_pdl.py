"""bench.py's sparse and dense steps (graph-captured, L2 flushed before each
replay) with SLSP_PDL=1 vs 0 in one process, round-robin (perf probing)."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

LAYERS = [("qkv", 4608, 3584), ("o", 3584, 3584), ("gate_up", 37888, 3584), ("down", 3584, 18944)]
M = 8192
g = torch.Generator(device="cuda").manual_seed(0)
Ls = []
for name, n, k in LAYERS:
    w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    pw = slsp.pack_compress(w, 6, 8)
    x = (torch.rand(M, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    Ls.append(dict(w=w, pw=pw, x=x, pay=torch.empty((M, pw.kp // 4), dtype=torch.int32, device="cuda"),
                   st=torch.empty(M, device="cuda"), q=torch.empty((M, k), dtype=torch.uint8, device="cuda"),
                   qs=torch.empty(M, device="cuda"), s_ch=torch.rand(n, device="cuda") * 0.01,
                   out=torch.empty((n, M), dtype=torch.bfloat16, device="cuda"), k=k))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def sparse_step():
    for L in Ls:
        slsp.fused_quant_slide(L["x"], 6, 8, check=False, payload=L["pay"], scales=L["st"])
        slsp.sparse_gemm(L["pw"], L["pay"], s_ch=L["s_ch"], s_tok=L["st"], out_mode=slsp.OUT_BF16_NM, out=L["out"])


def dense_step():
    for L in Ls:
        slsp.quantize_rows(L["x"], check=False, out=L["q"], scales=L["qs"])
        slsp.dense_gemm(L["w"], L["q"].view(torch.int8), s_ch=L["s_ch"], s_tok=L["qs"], out_mode=slsp.OUT_BF16_NM,
                        out=L["out"])


res = {}  # SLSP_PDL is read once per process by the library: run the script once per setting
pdl = os.environ.get("SLSP_PDL", "1")
for name, fn in (("sparse", sparse_step), ("dense", dense_step)):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[name] = (min(ts), statistics.median(ts))
print(f"PDL={pdl}: sparse step {res['sparse'][0]:.4f} (med {res['sparse'][1]:.4f}) ms | dense step "
      f"{res['dense'][0]:.4f} (med {res['dense'][1]:.4f}) ms | ratio {res['dense'][1] / res['sparse'][1]:.3f}")
