"""Measurements of BASELINE.json's other configs (GPU box; one JSON line per
case, then a markdown table). These are parity-test configs, not the bench
headline; bench.py measures configs[1]. Every timing: median of `reps`
launches, each after a 512 MiB L2-flush write, CUDA events on the stream.

  cfg1  6:8 INT8 K=N=4096, M=128: pack (offline), lift, sparse GEMM, plus the
        int32 result checked against dense_gemm on the quantized activations
  cfg3  Qwen2.5-7B shapes, 6:8 FP8 and the 4:6 / 8:10 INT8 patterns at
        M = 512 .. 16384: sparse GEMM vs the same-precision dense GEMM, against
        the bound N/(N-1) computed on the padded K'
  cfg4  Llama-3.1-8B shapes, 6:8 BF16, decode M = 1 / 16 / 64: sparse vs dense
        GEMM time and the weight-stream GB/s against HBM
  cfg5  Qwen2.5-14B 6:8 INT8 layer stack at M=8192, the per-GPU shard of an
        N-sharded run on 1/2/4/8 GPUs (one GPU here: the shard a rank owns)

  python tests/bench_configs.py [--cfg 1,3,4,5] [--reps 10] [--out profiles/r01_configs.md]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2603_05232_b200 as slsp  # noqa: E402

QWEN7 = [("qkv", 4608, 3584), ("o", 3584, 3584), ("gate_up", 37888, 3584), ("down", 3584, 18944)]
QWEN14 = [("qkv", 7168, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]
LLAMA8 = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
HBM = 6535.7
FLUSH = None


def timed(fn, reps):
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        FLUSH.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def gen():
    return torch.Generator(device="cuda").manual_seed(0)


def int8_weights(n, k, z, l, g):
    kk = -(-k // l) * l  # prune whole blocks, then cut to K (the tail block is zero-padded)
    w = torch.randint(-127, 128, (n, kk), dtype=torch.int8, device="cuda", generator=g)
    return slsp.magnitude_prune(w, z, l)[:, :k].contiguous()


def cfg1(reps, rows):
    n = k = 4096
    m = 128
    g = gen()
    w = int8_weights(n, k, 6, 8, g)
    x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    pw = slsp.pack_compress(w, 6, 8)
    t_pack = timed(lambda: slsp.pack_compress(w, 6, 8, check=False), reps)
    payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
    t_lift = timed(lambda: slsp.fused_quant_slide(x, 6, 8, check=False, payload=payload, scales=s_tok), reps)
    y = slsp.sparse_gemm(pw, payload)
    t_gemm = timed(lambda: slsp.sparse_gemm(pw, payload, out=y), reps)
    q, _ = slsp.quantize_rows(x)
    yd = slsp.dense_gemm(w, q.view(torch.int8))
    t_dense = timed(lambda: slsp.dense_gemm(w, q.view(torch.int8), out=yd), reps)
    exact = bool(torch.equal(y, yd))
    kp = pw.kp
    gemm_bytes = n * kp // 2 + n * kp // 8 + m * kp + n * m * 4
    rows.append({"cfg": 1, "case": "6:8 int8 4096x4096 M=128", "pack_us": t_pack * 1e3,
                 "pack_gbs": (n * k + n * kp // 2 + n * kp // 8) / t_pack / 1e6, "lift_us": t_lift * 1e3,
                 "gemm_us": t_gemm * 1e3, "gemm_gbs": gemm_bytes / t_gemm / 1e6, "dense_us": t_dense * 1e3,
                 "speedup": t_dense / t_gemm, "sparse_int32_equals_dense": exact})


def cfg3(reps, rows, ms):
    for z, l, kind in [(6, 8, "fp8"), (4, 6, "int8"), (8, 10, "int8")]:
        g = gen()
        for name, n, k in QWEN7:
            if kind == "fp8":
                wf = (torch.rand(n, -(-k // l) * l, device="cuda", generator=g) * 2 - 1) * 200
                w = slsp.magnitude_prune(wf.to(torch.float8_e4m3fn), z, l)[:, :k].contiguous()
            else:
                w = int8_weights(n, k, z, l, g)
            pw = slsp.pack_compress(w, z, l)
            qk = slsp.QUANT_FP8E4M3 if kind == "fp8" else slsp.QUANT_INT8
            s_ch = torch.rand(n, device="cuda", generator=g) * 0.01
            for m in ms:
                x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
                payload, s_tok = slsp.fused_quant_slide(x, z, l, kind=qk)
                q, q_s = slsp.quantize_rows(x, kind=qk)
                out = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
                t_s = timed(lambda: slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok,
                                                     out_mode=slsp.OUT_BF16_NM, out=out), reps)
                wd = w if kind == "int8" else w
                t_d = timed(lambda: slsp.dense_gemm(wd, q.view(w.dtype), s_ch=s_ch, s_tok=q_s,
                                                    out_mode=slsp.OUT_BF16_NM, out=out), reps)
                bound = 2 * k / pw.kp
                rows.append({"cfg": 3, "case": f"{z}:{l} {kind} {name} M={m}", "sparse_us": t_s * 1e3,
                             "dense_us": t_d * 1e3, "speedup": t_d / t_s, "bound": bound,
                             "sparse_eff_tflops": 2 * m * n * k / t_s / 1e9})
                del x, payload, q, out


def cfg4(reps, rows, ms):
    g = gen()
    for name, n, k in LLAMA8:
        w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16), 6, 8)
        pw = slsp.pack_compress(w, 6, 8)
        for m in ms:
            x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            lifted = slsp.lift_rows(x, 6, 8, kp=pw.kp)
            t_lift = timed(lambda: slsp.lift_rows(x, 6, 8, kp=pw.kp), reps)
            ys = slsp.sparse_gemm(pw, lifted)
            t_s = timed(lambda: slsp.sparse_gemm(pw, lifted, out=ys), reps)
            yd = slsp.dense_gemm(w, x)
            t_d = timed(lambda: slsp.dense_gemm(w, x, out=yd), reps)
            # the lift inside the GEMM (sparse_gemm_lift): the whole sparse step in one kernel
            yg = slsp.sparse_gemm_lift(pw, x)
            assert torch.equal(yg, ys), "sparse_gemm_lift != sparse_gemm(lift_rows)"
            t_g = timed(lambda: slsp.sparse_gemm_lift(pw, x, out=yg), reps)
            sb = n * pw.kp // 2 * 2 + n * pw.kp // 8 + m * pw.kp * 2 + n * m * 4
            gb = n * pw.kp // 2 * 2 + n * pw.kp // 8 + m * k * 2 + n * m * 4
            db = n * k * 2 + m * k * 2 + n * m * 4
            rows.append({"cfg": 4, "case": f"6:8 bf16 {name} M={m}", "lift_us": t_lift * 1e3, "sparse_us": t_s * 1e3,
                         "sparse_gbs": sb / t_s / 1e6, "sparse_hbm_frac": sb / t_s / 1e6 / HBM,
                         "glift_us": t_g * 1e3, "glift_hbm_frac": gb / t_g / 1e6 / HBM,
                         "dense_us": t_d * 1e3, "dense_gbs": db / t_d / 1e6, "speedup": t_d / t_s,
                         "step_speedup_glift": t_d / t_g, "bound": db / sb})


def cfg5(reps, rows):
    m = 8192
    g = gen()
    for gpus in (1, 2, 4, 8):
        tot_s = tot_d = 0.0
        for name, n, k in QWEN14:
            per = -(-n // gpus)
            per = -(-per // 128) * 128
            w = int8_weights(per, k, 6, 8, g)
            pw = slsp.pack_compress(w, 6, 8)
            x = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
            q, q_s = slsp.quantize_rows(x)
            s_ch = torch.rand(per, device="cuda", generator=g) * 0.01
            out = torch.empty((per, m), dtype=torch.bfloat16, device="cuda")
            tot_s += timed(lambda: (slsp.fused_quant_slide(x, 6, 8, check=False, payload=payload, scales=s_tok),
                                    slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok,
                                                     out_mode=slsp.OUT_BF16_NM, out=out)), reps)
            tot_d += timed(lambda: (slsp.quantize_rows(x, check=False, out=q, scales=q_s),
                                    slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=q_s,
                                                    out_mode=slsp.OUT_BF16_NM, out=out)), reps)
            del w, pw, x, payload, q, out
        flops = sum(2.0 * m * n * k for _, n, k in QWEN14)
        rows.append({"cfg": 5, "case": f"qwen2.5-14b 6:8 int8 stack, shard of {gpus} GPU(s)", "step_ms_per_gpu": tot_s,
                     "dense_step_ms_per_gpu": tot_d, "job_eff_tflops_if_linear": flops / (tot_s * 1e-3) / 1e12,
                     "speedup": tot_d / tot_s})


def cfg5s(reps, rows, nvlink_gbs=900.0):
    """Config 5 with the K-sharded lift, the per-GPU work of rank 0
    of G on one GPU: per layer the lift of its K/G column slice with the global
    |x|max (slsp_fused_quant_slide_scaled_multi, one destination — the local
    write; the G-1 peer copies are the same kernel's NVLink stores) + the GEMM
    of its N/G rows on the full payload. NVLink time = the slice's lifted bytes
    to G-1 peers at `nvlink_gbs` per direction; per-GPU step = sum over layers
    of max(lift, NVLink) + GEMM (the peer writes overlap the lift kernel)."""
    from paper_2603_05232_b200.sharding import lifted_col, shard_cols

    m = 8192
    g = gen()
    for gpus in (1, 2, 4, 8):
        tot = tot_lift = tot_gemm = tot_nv = 0.0
        for name, n, k in QWEN14:
            per = -(-n // gpus)
            per = -(-per // 128) * 128
            w = int8_weights(per, k, 6, 8, g)
            pw = slsp.pack_compress(w, 6, 8)
            k0, k1 = shard_cols(k, gpus, 0)
            x = (torch.rand(m, k1 - k0, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            amax = slsp.row_absmax(x)
            payload = torch.zeros((m, pw.kp // 4), dtype=torch.int32, device="cuda")
            scales = torch.empty(m, device="cuda")
            s_ch = torch.rand(per, device="cuda", generator=g) * 0.01
            out = torch.empty((per, m), dtype=torch.bfloat16, device="cuda")
            t_l = timed(lambda: slsp.fused_quant_slide_multi(x, 6, 8, amax, [payload], pw.kp, lifted_col(k0, 6, 8),
                                                             scales=scales, check=False), reps)
            payload.slsp_kind, payload.slsp_pattern = slsp.QUANT_INT8, (6, 8)
            t_g = timed(lambda: slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=scales, out_mode=slsp.OUT_BF16_NM,
                                                 out=out), reps)
            nv_ms = m * (k1 - k0) * 1.5 * (gpus - 1) / (nvlink_gbs * 1e6)
            tot_lift += t_l
            tot_gemm += t_g
            tot_nv += nv_ms
            tot += max(t_l, nv_ms) + t_g
            del w, pw, x, payload, out
        flops = sum(2.0 * m * n * k for _, n, k in QWEN14)
        rows.append({"cfg": 5, "case": f"qwen2.5-14b 6:8 int8 stack, K-sharded lift, rank 0 of {gpus}",
                     "step_ms_per_gpu": tot, "lift_ms": tot_lift, "gemm_ms": tot_gemm, "nvlink_ms_projected": tot_nv,
                     "job_eff_tflops_if_linear": flops / (tot * 1e-3) / 1e12})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="1,3,4,5")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ms3", default="512,2048,8192,16384")
    ap.add_argument("--ms4", default="1,16,64")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = []
    sel = {int(c) for c in a.cfg.split(",")}
    if 1 in sel:
        cfg1(a.reps, rows)
    if 3 in sel:
        cfg3(a.reps, rows, [int(v) for v in a.ms3.split(",")])
    if 4 in sel:
        cfg4(a.reps, rows, [int(v) for v in a.ms4.split(",")])
    if 5 in sel:
        cfg5(a.reps, rows)
        cfg5s(a.reps, rows)
    for r in rows:
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    if a.out:
        keys = []
        for r in rows:
            keys += [k for k in r if k not in keys]
        lines = ["| " + " | ".join(keys) + " |", "|" + "---|" * len(keys)]
        for r in rows:
            cells = []
            for k in keys:
                v = r.get(k, "")
                cells.append(f"{v:.3f}" if isinstance(v, float) else str(v))
            lines.append("| " + " | ".join(cells) + " |")
        Path(a.out).write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
