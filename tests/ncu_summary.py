"""Summarise ncu captures for profiles/ (run here, on the .ncu-rep files that
gpurun brought back).

    python tests/ncu_summary.py gpurun_out/prof_sgemm.ncu-rep ... > profiles/rNN_ncu_full.txt
    python tests/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rNN_launches_summary.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "kernel time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM bytes"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "L2->SM rate"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed", "L2->SM % of peak"),
    ("lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "L2 slice (tex) % of peak"),
    ("lts__t_sectors_srcunit_ltcfabric.avg.pct_of_peak_sustained_elapsed", "L2 cross-die fabric % of peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (non-realtime)"),
    ("sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "UMA (tcgen05) pipe inst % of peak"),
    ("sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active", "TMA pipe inst % of peak"),
]


def grep(paths, pattern):
    """Every raw metric whose name matches `pattern` (regex), per capture."""
    import re

    rx = re.compile(pattern)
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        head, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"== {path.split('/')[-1]}: {r[head.index('Kernel Name')][:100]}")
            for i, h in enumerate(head):
                if rx.search(h):
                    print(f"   {h:90s} {r[i]:>16s} {units[i]}")


def full(paths):
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        head, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"== {path.split('/')[-1]}")
            print(f"   kernel: {r[head.index('Kernel Name')][:160]}")
            for name, label in METRICS:
                if name in head:
                    i = head.index(name)
                    print(f"   {label:32s} {r[i]:>14s} {units[i]:10s} ({name})")
            dr = [r[head.index(m)] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum") if m in head]
            print()


def launches(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    per = defaultdict(list)
    for r in csv.DictReader(io.StringIO(text)):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0][:110] if "slsp" in name or "gemm_kernel" in name or "kernel<" in name else name[:60]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
        per[short].append(float(r["Metric Value"].replace(",", "")) * scale)
    total = sum(sum(v) for v in per.values())
    print(f"{'kernel':112s} {'launches':>8s} {'avg us':>9s} {'total us':>10s} {'share':>6s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:112s} {len(v):8d} {sum(v) / len(v):9.1f} {sum(v):10.1f} {sum(v) / total:6.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--grep":
        grep(sys.argv[3:], sys.argv[2])
    else:
        full(sys.argv[1:])
