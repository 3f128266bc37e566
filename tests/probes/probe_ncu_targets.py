"""Minimal ncu targets (GPU box; perf probing): runs one op 4 times after L2
flushes. Modes: cfg1_sparse / cfg1_dense (6:8 INT8 4096x4096, M=128),
dec_sparse / dec_dense (Llama-3.1-8B qkv 6144x4096 BF16, M=1), lift_m1 /
lift_m8192 (fused_quant_slide of a 3584-wide BF16 X), glift_mM / gsparse_mM
(gate_up 28672x4096 BF16: sparse_gemm_lift vs sparse_gemm on lifted rows), chain_amax (sparse GEMM
o_proj 3584x3584 M=8192 MN with the token |y|max fold)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

mode = sys.argv[1]
g = torch.Generator(device="cuda").manual_seed(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
if mode.startswith("cfg1"):
    w = slsp.magnitude_prune(torch.randint(-127, 128, (4096, 4096), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(128, 4096, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    pay, st = slsp.fused_quant_slide(x, 6, 8, kp=pw.kp)
    q, qs = slsp.quantize_rows(x)
    fn = (lambda: slsp.sparse_gemm(pw, pay)) if mode == "cfg1_sparse" else (lambda: slsp.dense_gemm(w, q.view(torch.int8)))
elif mode.startswith("dec"):
    w = slsp.magnitude_prune((torch.rand(6144, 4096, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
    x = (torch.rand(1, 4096, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    lifted = slsp.lift_rows(x, 6, 8, kp=pw.kp)
    fn = (lambda: slsp.sparse_gemm(pw, lifted)) if mode == "dec_sparse" else (lambda: slsp.dense_gemm(w, x))
elif mode.startswith("glift") or mode.startswith("gsparse"):
    m = int(mode.split("_m")[1])  # Llama-3.1-8B gate_up BF16: in-GEMM lift vs lifted operand
    w = slsp.magnitude_prune((torch.rand(28672, 4096, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
    x = (torch.rand(m, 4096, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    lifted = slsp.lift_rows(x, 6, 8, kp=pw.kp)
    fn = (lambda: slsp.sparse_gemm_lift(pw, x)) if mode.startswith("glift") else (lambda: slsp.sparse_gemm(pw, lifted))
elif mode.startswith("lift"):
    m = int(mode.split("_m")[1])
    if mode.startswith("liftg"):  # gaussian rows with per-row scales (absmax not a power of two)
        x = (torch.randn(m, 3584, device="cuda", generator=g) * (torch.rand(m, 1, device="cuda", generator=g) * 3 + 0.1)).to(torch.bfloat16)
    else:
        x = (torch.rand(m, 3584, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pay, st = slsp.fused_quant_slide(x, 6, 8)
    fn = lambda: slsp.fused_quant_slide(x, 6, 8, check=False, payload=pay, scales=st)  # noqa: E731
elif mode == "chain_amax":
    w = slsp.magnitude_prune(torch.randint(-127, 128, (3584, 3584), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    x = (torch.rand(8192, 3584, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    pay, st = slsp.fused_quant_slide(x, 6, 8)
    s_ch = torch.rand(3584, device="cuda", generator=g) * 0.01
    am = torch.empty(8192, device="cuda")
    fn = lambda: slsp.sparse_gemm(pw, pay, s_ch=s_ch, s_tok=st, out_mode=slsp.OUT_BF16_MN, tok_amax=am)  # noqa: E731
else:
    raise SystemExit(f"unknown mode {mode}")
for _ in range(4):
    flush.zero_()
    fn()
torch.cuda.synchronize()
print("ok", mode)
