"""Summarise ncu captures into profiles/ (tracked evidence).

  python tools/ncu_summary.py --rep gpurun_out/prof_r1.ncu-rep \
      --launches gpurun_out/launches_bench.csv --out profiles/round1

Writes <out>/ncu_summary.json (per tensor-core kernel: duration, DRAM bytes,
tensor-pipe activity, SM clock, top stall reasons), <out>/launches.md (the
serialised launch list of one bench step) and profiles/ncu_summary.json (the
per-launch DRAM traffic bench.py reports as roofline.traffic).
"""

import argparse
import csv
import io
import json
import os
import subprocess

KERNEL_KEYS = [  # order of the tensor-core launches within one step
    ("logits_kernel<2", "logits_fwd"),    # forward + E store (canonical shapes)
    ("logits_kernel<0", "logits_fwd"),    # forward only (recompute path)
    ("logits_kernel<1", "logits_grad"),   # recompute path only
    ("gemm_kernel", "gemm_backward"),     # single rank: intra + cross in one launch
]
MULTI_RANK_GEMMS = [("gemm_kernel", "gemm_cross"), ("gemm_kernel", "gemm_intra")]
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "lts__t_sector_op_read_hit_rate.pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "launch__grid_size",
    "launch__cluster_dim_x",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
]
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
              "ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9,
              "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def value(h, units, r, key):
    if key not in h:
        return None
    i = h.index(key)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return r[i]
    return v * UNIT_SCALE.get(units[i], 1.0)


def summarize_rep(rep):
    h, units, rows = raw_rows(rep)
    stall_keys = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    out = {}
    seen = {}
    for r in rows:
        name = r[h.index("Kernel Name")].replace("(int)", "")
        for pat, key in KERNEL_KEYS:
            if pat in name:
                n = seen.get(pat, 0)
                keys = [k for p, k in KERNEL_KEYS if p == pat]
                if n < len(keys) and keys[n] not in out:
                    k = keys[n]
                    seen[pat] = n + 1
                    m = {mk: value(h, units, r, mk) for mk in METRICS}
                    stalls = sorted(((sk.replace("smsp__pcsamp_warps_issue_stalled_", ""), value(h, units, r, sk) or 0.0)
                                     for sk in stall_keys), key=lambda x: -x[1])[:6]
                    m["top_stalls"] = stalls
                    m["kernel_name"] = name
                    m["dram_bytes_per_launch"] = (m["dram__bytes_read.sum"] or 0) + (m["dram__bytes_write.sum"] or 0)
                    out[k] = m
                break
    return out


def launches_md(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    lines = ["| # | kernel | time (us) |", "|---|---|---|"]
    total = 0.0
    n = 0
    for r in rows[hi + 1:]:
        if "disco" not in r[ki]:
            continue
        t = float(r[vi].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        lines.append(f"| {n} | `{r[ki][:70]}` | {t:.1f} |")
        total += t
        n += 1
    lines.append(f"| | total ({n} disco launches) | {total:.1f} |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--multi-rank", action="store_true", help="separate cross / intra GEMM launches (N > 1)")
    a = ap.parse_args()
    if a.multi_rank:
        KERNEL_KEYS[:] = [k for k in KERNEL_KEYS if k[0] != "gemm_kernel"] + MULTI_RANK_GEMMS
    os.makedirs(a.out, exist_ok=True)
    summ = summarize_rep(a.rep)
    with open(os.path.join(a.out, "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    root = os.path.dirname(os.path.abspath(a.out.rstrip("/")))
    with open(os.path.join(root, "ncu_summary.json"), "w") as f:
        json.dump({k: v["dram_bytes_per_launch"] for k, v in summ.items()}, f, indent=1)
    if a.launches:
        with open(os.path.join(a.out, "launches.md"), "w") as f:
            f.write("Serialised launch list (ncu --metrics gpu__time_duration.sum --clock-control none), "
                    "cold caches: compare shares, not absolutes.\n\n")
            f.write(launches_md(a.launches) + "\n")
    for k, v in summ.items():
        print(f"{k:12s} {v['gpu__time_duration.sum'] * 1e3:8.3f} ms  dram {v['dram_bytes_per_launch'] / 1e9:6.2f} GB  "
              f"tensor {v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:5.1f}%  "
              f"sm {v['sm__cycles_elapsed.avg.per_second'] / 1e9:.2f} GHz")


if __name__ == "__main__":
    main()
