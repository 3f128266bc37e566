"""GEMM config sweep in ONE process (GPU box; perf probing, not a test).

Each config is applied by setting os.environ + slsp.reload_knobs() before
capturing a CUDA graph of `reps` launches. Prints one
line per (kernel, config, layer): ms per launch (median of `rounds` graph
replays, CUDA events) and effective TFLOPS; sparse/dense ratios at the end.

  python tests/probe_sweep.py [--layers gate_up,down] [--sparse 'MSUB=2 CLUSTER=2;MSUB=1']
                              [--dense 'CLUSTER=2;CLUSTER=4'] [--reps 10] [--rounds 5]
Sparse keys map to SLSP_GEMM_<KEY>, dense keys to SLSP_DGEMM_<KEY> (CLUSTER,
MSUB) or SLSP_GEMM_<KEY> (GROUP, HINTS, DEBUG, ...).
"""
import argparse
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_05232_b200 as slsp  # noqa: E402

SHAPES = {"qkv": (4608, 3584), "o": (3584, 3584), "gate_up": (37888, 3584), "down": (3584, 18944),
          "cfg1": (4096, 4096),
          # L2-residency probes: gate_up's K with fewer weight rows (operands fit in L2)
          "gu4k": (4096, 3584), "gu8k": (8192, 3584), "gu16k": (16384, 3584),
          # BASELINE config 5: Qwen2.5-14B row shards of 8 GPUs (rounded up to 128 rows)
          "qkv14s8": (896, 5120), "o14s8": (640, 5120), "gu14s8": (3456, 5120), "down14s8": (640, 13824)}  # BASELINE config 1 (K = N = 4096)
DENSE_KEYS = {"CLUSTER", "MSUB", "DECODE_M"}


def parse_cfgs(s):
    out = []
    for part in s.split(";"):
        kv = dict(x.split("=") for x in part.split() if "=" in x)
        out.append(kv)
    return out


def apply(kv, dense):
    for k in list(os.environ):
        if k.startswith("SLSP_GEMM_") or k.startswith("SLSP_DGEMM_"):
            del os.environ[k]
    for k, v in kv.items():
        pre = "SLSP_DGEMM_" if dense and k in DENSE_KEYS else "SLSP_GEMM_"
        os.environ[pre + k] = v
    slsp.reload_knobs()  # the library snapshots SLSP_* knobs


class Clocks:
    """NVML SM-clock / power sampler around a timed region."""

    def __init__(self):
        import threading

        import pynvml

        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.samples = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
            self.stop.wait(0.002)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join()

    def summary(self):
        if not self.samples:
            return "clk ? pw ?"
        c = sorted(s[0] for s in self.samples)
        p = sorted(s[1] for s in self.samples)
        return f"clk {c[len(c) // 2]:4d} pw {p[len(p) // 2]:4.0f}W"


FLUSH = None
FLUSH_READ = None
BURST = False
CLEAN = False  # after the flush write, read another >L2 buffer so L2 holds clean lines


def timeit_burst(fn, reps, rounds):
    """bench.py's regime: each launch alone after a 512 MiB L2-flush write."""
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    global FLUSH_READ
    if CLEAN and FLUSH_READ is None:
        FLUSH_READ = torch.ones(256 << 20, dtype=torch.int32, device="cuda")
    fn()
    torch.cuda.synchronize()
    evs = []
    clk = Clocks()
    with clk:
        for _ in range(reps):
            FLUSH.zero_()
            if CLEAN:
                FLUSH_READ.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
    timeit_burst.clk = clk.summary()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def timeit(fn, reps, rounds):
    if BURST:
        r = timeit_burst(fn, reps, rounds)
        timeit.clk = timeit_burst.clk
        return r
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    clk = Clocks()
    with clk:
        for _ in range(rounds):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / reps)
    timeit.clk = clk.summary()
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="gate_up,down,qkv,o")
    ap.add_argument("--sparse", default="")
    ap.add_argument("--dense", default="")
    ap.add_argument("--sparsex", default="", help="configs of the in-SM-lifting kernel (sparse_gemm_x)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cycles", type=int, default=3, help="round-robin passes over the configs (min reported)")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--cublas", action="store_true", help="also time torch._int_mm (cuBLASLt int8)")
    ap.add_argument("--clean", action="store_true", help="burst: read a 1 GiB buffer after the flush write")
    ap.add_argument("--lift", action="store_true", help="also time fused_quant_slide / quantize_rows")
    ap.add_argument("--mn", action="store_true", help="token-major [M][N] output")
    ap.add_argument("--burst", action="store_true", help="bench.py regime: single launches after L2 flushes")
    ap.add_argument("--check", action="store_true", help="compare each sparse config's int32 output with the first")
    ap.add_argument("--bf16", action="store_true", help="BF16 weights/activations (kind f16) instead of INT8")
    a = ap.parse_args()
    global BURST, CLEAN
    BURST = a.burst
    CLEAN = a.clean
    m = a.m
    best = {}
    for layer in a.layers.split(","):
        n, k = SHAPES[layer]
        gen = torch.Generator(device="cuda").manual_seed(0)
        x = (torch.rand(m, k, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)
        if a.bf16:
            w = slsp.magnitude_prune((torch.rand(n, k, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16), 6, 8)
            pw = slsp.pack_compress(w, 6, 8)
            payload, s_tok = slsp.lift_rows(x, 6, 8, kp=pw.kp), None
            q, q_s = x, None
            s_ch = None
        else:
            w = slsp.magnitude_prune(torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=gen),
                                     6, 8)
            pw = slsp.pack_compress(w, 6, 8)
            payload, s_tok = slsp.fused_quant_slide(x, 6, 8)
            q, q_s = slsp.quantize_rows(x)
            s_ch = torch.rand(n, device="cuda") * 0.01
        out = torch.empty((m, n) if a.mn else (n, m), dtype=torch.bfloat16, device="cuda")
        om = slsp.OUT_BF16_MN if a.mn else slsp.OUT_BF16_NM
        if a.bf16:  # no scales: fp32 accumulators out
            out, om = torch.empty((n, m), dtype=torch.float32, device="cuda"), slsp.OUT_RAW_NM
        flops = 2.0 * m * n * k
        ref = None
        if a.lift:
            kb = m * (2 * k + pw.kp + 4)
            ms = timeit(lambda: slsp.fused_quant_slide(x, 6, 8, check=False, payload=payload, scales=s_tok), a.reps, a.rounds)
            print(f"lift   {layer:8s} {'fused_quant_slide 6:8 int8':40s} {ms:8.4f} ms {kb / ms / 1e6:8.1f} GB/s {timeit.clk}")
            kb = m * (2 * k + q.shape[1] + 4)
            ms = timeit(lambda: slsp.quantize_rows(x, check=False, out=q, scales=q_s), a.reps, a.rounds)
            print(f"quant  {layer:8s} {'quantize_rows int8':40s} {ms:8.4f} ms {kb / ms / 1e6:8.1f} GB/s {timeit.clk}")
        if a.cublas:  # library reference point: cuBLASLt int8 GEMM (int32 out) via torch._int_mm
            xq = q.view(torch.int8)[:, :k].contiguous()
            try:
                ms = timeit(lambda: torch._int_mm(xq, w.t()), a.reps, a.rounds)
                print(f"cublas {layer:8s} {'torch._int_mm int8->int32':40s} {ms:8.4f} ms {flops / ms / 1e9:8.1f} TFLOPS "
                      f"{timeit.clk}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"cublas {layer:8s} ERROR {e}", flush=True)
        runs = []  # (kind, kv, fn)
        if a.sparsex:
            xq, _ = slsp.quantize_rows(x, kpad=slsp.round_up(k, 512))
            pw.gemm_order()
        for kind, cfgs in (("sparse", a.sparse), ("sparsex", a.sparsex), ("dense", a.dense)):
            if not cfgs:
                continue
            for kv in parse_cfgs(cfgs):
                if kind == "sparsex":
                    fn = lambda: slsp.sparse_gemm_x(pw, xq, s_ch=s_ch, s_tok=s_tok, out_mode=om, out=out)
                elif kind == "sparse":
                    fn = lambda: slsp.sparse_gemm(pw, payload, s_ch=s_ch, s_tok=s_tok, out_mode=om, out=out)
                else:
                    fn = lambda: slsp.dense_gemm(w, q if a.bf16 else q.view(torch.int8), s_ch=s_ch, s_tok=q_s,
                                                 out_mode=om, out=out)
                runs.append((kind, kv, fn))
        # round-robin over the configs so every config sees the same thermal/power history
        res = {i: [] for i in range(len(runs))}
        for _ in range(a.cycles):
            for i, (kind, kv, fn) in enumerate(runs):
                apply(kv, kind == "dense")
                try:
                    res[i].append(timeit(fn, a.reps, a.rounds))
                except Exception as e:  # noqa: BLE001
                    print(f"{kind:6s} {layer:8s} {str(kv):40s} ERROR {e}", flush=True)
                    res[i].append(float("inf"))
        for i, (kind, kv, fn) in enumerate(runs):
            apply(kv, kind == "dense")
            tag = ""
            if a.check and kind.startswith("sparse") and not kv.get("DEBUG"):
                y = (slsp.sparse_gemm(pw, payload) if kind == "sparse" else slsp.sparse_gemm_x(pw, xq)).clone()
                if ref is None:
                    ref = y
                tag = " ok" if torch.equal(y, ref) else " MISMATCH"
            ms = min(res[i])
            med = statistics.median(res[i])
            print(f"{kind:6s} {layer:8s} {str(kv):40s} {ms:8.4f} ms (med {med:.4f}) {flops / ms / 1e9:8.1f} TFLOPS{tag}",
                  flush=True)
            key = (kind, layer)
            if key not in best or ms < best[key][0]:
                best[key] = (ms, kv)
        apply({}, False)
    for layer in a.layers.split(","):
        for sk in ("sparse", "sparsex"):
            if (sk, layer) in best and ("dense", layer) in best:
                s, d = best[(sk, layer)], best[("dense", layer)]
                print(f"best {layer}: {sk} {s[0]:.4f} {s[1]}  dense {d[0]:.4f} {d[1]}  x{d[0] / s[0]:.3f}")


if __name__ == "__main__":
    main()
