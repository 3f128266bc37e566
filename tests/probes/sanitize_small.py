"""Small-shape run of every kernel family for compute-sanitizer (GPU box):
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tests/probes/sanitize_small.py
Covers: packers (6:8 LUT byte path, generic patterns, bf16), magnitude_prune,
lift (row-resident, warp, generic, scaled, multi-destination), quantize_rows,
row_absmax, sparse GEMM configs (int8 two-subtile / one-subtile / 256-token /
decode split-K, FP8, BF16, both output layouts, amax fold, in-SM lifting),
dense GEMM (int8, FP8, BF16, decode split-K), the in-GEMM BF16 lift. Prints one line per step."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402


def step(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    n, k = 512, 1024
    w8 = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g), 6, 8)
    wb = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) - 0.5).to(torch.bfloat16), 6, 8)
    wf = slsp.magnitude_prune(((torch.rand(n, k, device="cuda", generator=g) - 0.5) * 100).to(torch.float8_e4m3fn), 6, 8)
    s_ch = torch.rand(n, device="cuda", generator=g) * 0.01
    step("pack 6:8 int8", lambda: slsp.pack_compress(w8, 6, 8))
    step("pack 4:6 int8", lambda: slsp.pack_compress(slsp.magnitude_prune(w8[:, :960].contiguous(), 4, 6), 4, 6))
    step("pack 6:8 bf16", lambda: slsp.pack_compress(wb, 6, 8))
    step("pack_matrix", lambda: slsp.pack_matrix(w8, 6, 8))
    p8, pb, pf = slsp.pack_compress(w8, 6, 8), slsp.pack_compress(wb, 6, 8), slsp.pack_compress(wf, 6, 8)
    for m, tag in [(8192 // 8, "M=1024"), (300, "M=300"), (64, "decode M=64"), (1, "M=1")]:
        x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        step(f"lift {tag}", lambda: slsp.fused_quant_slide(x, 6, 8))
        step(f"lift fp32 warp path {tag}", lambda: slsp.fused_quant_slide(x.float(), 6, 8))
        step(f"lift 4:6 {tag}", lambda: slsp.fused_quant_slide(x[:, :960].contiguous(), 4, 6))
        step(f"quantize_rows {tag}", lambda: slsp.quantize_rows(x))
        step(f"row_absmax {tag}", lambda: slsp.row_absmax(x))
        pay, st = slsp.fused_quant_slide(x, 6, 8, kp=p8.kp)
        q, qs = slsp.quantize_rows(x)
        a = slsp.row_absmax(x)
        step(f"lift scaled {tag}", lambda: slsp.fused_quant_slide(x, 6, 8, kp=p8.kp, absmax=a))
        bufs = [torch.zeros((m, p8.kp // 4), dtype=torch.int32, device="cuda") for _ in range(2)]
        step(f"lift multi {tag}", lambda: slsp.fused_quant_slide_multi(x[:, 512:].contiguous(), 6, 8, a, bufs, p8.kp,
                                                                       768))
        for om, on in [(slsp.OUT_RAW_NM, "raw"), (slsp.OUT_BF16_NM, "nm"), (slsp.OUT_BF16_MN, "mn")]:
            for msub in ("1", "2"):
                os.environ["SLSP_GEMM_MSUB"] = msub
                slsp.reload_knobs()
                step(f"sparse int8 {tag} {on} msub{msub}",
                     lambda: slsp.sparse_gemm(p8, pay, s_ch=s_ch, s_tok=st, out_mode=om))
            os.environ.pop("SLSP_GEMM_MSUB")
            slsp.reload_knobs()
            step(f"dense int8 {tag} {on}", lambda: slsp.dense_gemm(w8, q.view(torch.int8), s_ch=s_ch, s_tok=qs,
                                                                   out_mode=om))
        am = torch.empty(m, device="cuda")
        step(f"sparse amax fold {tag} mn", lambda: slsp.sparse_gemm(p8, pay, s_ch=s_ch, s_tok=st,
                                                                   out_mode=slsp.OUT_BF16_MN, tok_amax=am))
        step(f"sparse amax fold {tag} nm", lambda: slsp.sparse_gemm(p8, pay, s_ch=s_ch, s_tok=st,
                                                                   out_mode=slsp.OUT_BF16_NM, tok_amax=am))
        payf, stf = slsp.fused_quant_slide(x, 6, 8, kind=slsp.QUANT_FP8E4M3, kp=pf.kp)
        qf, qfs = slsp.quantize_rows(x, kind=slsp.QUANT_FP8E4M3)
        step(f"sparse fp8 {tag}", lambda: slsp.sparse_gemm(pf, payf, s_ch=s_ch, s_tok=stf, out_mode=slsp.OUT_BF16_NM))
        step(f"dense fp8 {tag}", lambda: slsp.dense_gemm(wf, qf.view(torch.float8_e4m3fn), s_ch=s_ch, s_tok=qfs,
                                                         out_mode=slsp.OUT_BF16_NM))
        lifted = slsp.lift_rows(x, 6, 8, kp=pb.kp)
        step(f"sparse bf16 {tag}", lambda: slsp.sparse_gemm(pb, lifted))
        step(f"dense bf16 {tag}", lambda: slsp.dense_gemm(wb, x))
        step(f"sparse bf16 in-GEMM lift {tag}", lambda: slsp.sparse_gemm_lift(pb, x, s_ch=s_ch, s_tok=st,
                                                                            out_mode=slsp.OUT_BF16_NM))
        xs = torch.zeros((m, k + 2), dtype=torch.bfloat16, device="cuda")[:, :k]  # 4-byte path
        step(f"sparse bf16 in-GEMM lift strided {tag}", lambda: slsp.sparse_gemm_lift(pb, xs))
        if m >= 64:
            xq, _ = slsp.quantize_rows(x, kpad=slsp.round_up(k, 512))
            step(f"sparse in-SM lift {tag}", lambda: slsp.sparse_gemm_x(p8, xq))


if __name__ == "__main__":
    main()
