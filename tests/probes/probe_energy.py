"""Energy per launch of GEMM configs under sustained load (GPU box; perf probing).

Each config runs back to back for `--seconds` (CUDA-graph replays of 20
launches) while NVML samples SM clock / power / throttle reasons every 5 ms;
the board energy counter (nvmlDeviceGetTotalEnergyConsumption, mJ) is read
around the timed region. Prints per config: ms per launch, median SM clock,
median power, joules per launch and effective TOP/J. Under the board power
cap the clock settles where power = cap, so time per launch ~ energy per
launch / cap: the kernel that needs fewer joules per effective op is the
faster one regardless of its cycle efficiency.

  python tests/probes/probe_energy.py --layers gate_up --sparse 'MSUB=2;MSUB=2 DEBUG=3' --dense 'CLUSTER=2'
"""
import argparse
import json
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_2603_05232_b200 as slsp  # noqa: E402
from probe_sweep import SHAPES, apply, parse_cfgs  # noqa: E402


def sampler(stop, out, nv, h):
    while not stop.is_set():
        out.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.005)


def run(nv, h, name, fn, ops, seconds):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    g.replay()
    torch.cuda.synchronize()
    time.sleep(0.3)  # let the board cool to a comparable starting point
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(stop, samples, nv, h))
    th.start()
    e_a = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    reps = 0
    while time.time() - t0 < seconds:
        g.replay()
        reps += 20
        if reps % 200 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    e_b = nv.nvmlDeviceGetTotalEnergyConsumption(h)
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    busy = [s for s in samples if s[1] > 300]
    clk = sorted(s[0] for s in busy) or [0]
    pw = sorted(s[1] for s in busy) or [0]
    reasons = 0
    for s in busy:
        reasons |= s[2]
    joules = (e_b - e_a) / 1000.0 / reps
    rec = {"kernel": name, "ms": round(ms, 4), "tops": round(ops / ms / 1e9, 1), "sm_mhz": clk[len(clk) // 2],
           "power_w": round(pw[len(pw) // 2], 1), "j_per_launch": round(joules, 5),
           "top_per_j": round(ops / joules / 1e12, 2) if joules > 0 else None, "reasons": hex(reasons),
           "samples": len(busy)}
    print(json.dumps(rec), flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="gate_up")
    ap.add_argument("--sparse", default="MSUB=2")
    ap.add_argument("--dense", default="CLUSTER=2")
    ap.add_argument("--sparsex", default="", help="configs of the in-SM-lifting kernel (sparse_gemm_x)")
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--m", type=int, default=8192)
    args = ap.parse_args()
    import pynvml as nv

    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    m = args.m
    for layer in args.layers.split(","):
        n, k = SHAPES[layer]
        gen = torch.Generator(device="cuda").manual_seed(0)
        w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=gen), 6, 8)
        x = (torch.rand(m, k, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)
        pw = slsp.pack_compress(w, 6, 8)
        payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
        q, q_s = slsp.quantize_rows(x)
        s_ch = torch.rand(n, device="cuda") * 0.01
        out = torch.empty((n, m), dtype=torch.bfloat16, device="cuda")
        ops = 2.0 * m * n * k
        for kv in parse_cfgs(args.sparse) if args.sparse else []:
            apply(kv, False)
            run(nv, h, f"sparse {layer} {kv}", lambda: slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok,
                                                                         out_mode=slsp.OUT_BF16_NM, out=out),
                ops, args.seconds)
        if args.sparsex:
            xq, _ = slsp.quantize_rows(x, kpad=slsp.round_up(k, 512))
            pwx = pw.gemm_order()
        for kv in parse_cfgs(args.sparsex) if args.sparsex else []:
            apply(kv, False)
            run(nv, h, f"sparsex {layer} {kv}", lambda: slsp.sparse_gemm_x(pwx, xq, s_ch=s_ch, s_tok=s_tok,
                                                                            out_mode=slsp.OUT_BF16_NM, out=out),
                ops, args.seconds)
        for kv in parse_cfgs(args.dense) if args.dense else []:
            apply(kv, True)
            run(nv, h, f"dense {layer} {kv}", lambda: slsp.dense_gemm(w, q.view(torch.int8), s_ch=s_ch, s_tok=q_s,
                                                                       out_mode=slsp.OUT_BF16_NM, out=out),
                ops, args.seconds)
        apply({}, False)


if __name__ == "__main__":
    main()
