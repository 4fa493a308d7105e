"""Summarise ncu outputs into profiles/ (run in the build container, no GPU needed).

  python scripts/summarize_ncu.py launches <launches.csv> [top]   -> per-kernel time shares
  python scripts/summarize_ncu.py kernel <report.ncu-rep> <regex>  -> key metrics per launch
"""

from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum"]


def launches(path: str, top: int = 25) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki])[:100]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"launches: {sum(cnt.values())}, total device time {T / 1e3:.1f} ms (serialised, cold cache)",
           "", "| share | time (us) | launches | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"| {v / T * 100:.2f}% | {v:.0f} | {cnt[k]} | `{k}` |")
    mine = sum(v for k, v in tot.items()
               if any(t in k for t in ("zi::", "fused::", "gemm", "gsk::", "attn::", "emb::")) or
               k.startswith(("rs_kernel", "adam_kernel", "gather_", "linear_fwd")))
    lib = sum(v for k, v in tot.items() if "nvjet" in k or "cudnn" in k or "cutlass" in k)
    other = T - mine - lib
    out.append("")
    out.append(f"libzinf kernels: {mine / T * 100:.2f}% of device time; cuBLAS / cuDNN: "
               f"{lib / T * 100:.2f}%; other (torch elementwise glue): {other / T * 100:.2f}%")
    return "\n".join(out)


def kernel(report: str, regex: str) -> str:
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    out = ["| metric | unit | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |",
           "|---|---|" + "---:|" * (len(rows) - 2)]
    sel = [r for r in rows[2:] if re.search(regex, r[ki])]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            out.append(f"| {k} | {units[i]} | " + " | ".join(r[i] for r in sel) + " |")
    names = sorted({re.sub(r"\(.*", "", r[ki]) for r in sel})
    return f"kernel: {', '.join(names)}\n\n" + "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25))
    else:
        print(kernel(sys.argv[2], sys.argv[3]))
