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


def launches_md(path, hbm_gbs=None):
    """Launch list of one step from an ncu metrics CSV (one row per kernel x metric): duration and,
    when captured, DRAM bytes -> achieved GB/s per launch (the HBM side of the elementwise tails)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ii, ki, mi, vi, ui = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), \
        h.index("Metric Unit")
    launches = {}
    order = []
    for r in rows[hi + 1:]:
        if "disco" not in r[ki]:
            continue
        if r[ii] not in launches:
            launches[r[ii]] = {"name": r[ki]}
            order.append(r[ii])
        launches[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1.0)
    lines = ["| # | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | GB/s |", "|---|---|---|---|---|---|"]
    total = 0.0
    table = []
    for n, key in enumerate(order):
        L = launches[key]
        t = L.get("gpu__time_duration.sum", 0.0)
        rd, wr = L.get("dram__bytes_read.sum"), L.get("dram__bytes_write.sum")
        gbs = (rd + wr) / t / 1e9 if (rd is not None and wr is not None and t > 0) else None
        lines.append(f"| {n} | `{L['name'][:70]}` | {t * 1e6:.1f} | "
                     f"{'' if rd is None else f'{rd / 1e6:.1f}'} | {'' if wr is None else f'{wr / 1e6:.1f}'} | "
                     f"{'' if gbs is None else f'{gbs:.0f}'} |")
        table.append({"kernel": L["name"][:90], "us": t * 1e6, "dram_read_mb": None if rd is None else rd / 1e6,
                      "dram_write_mb": None if wr is None else wr / 1e6, "gbs": gbs,
                      "frac_of_hbm": (gbs / hbm_gbs) if (gbs and hbm_gbs) else None})
        total += t
    lines.append(f"| | total ({len(order)} disco launches) | {total * 1e6:.1f} | | | |")
    return "\n".join(lines), table


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
        hbm = None
        peaks = os.path.join(os.path.dirname(root), "MEASURED_PEAKS.json")
        if os.path.exists(peaks):
            try:
                pk = json.load(open(peaks))
                hbm = pk.get("hbm_copy_gbs") or pk.get("hbm_gbs")
            except Exception:
                hbm = None
        md, table = launches_md(a.launches, hbm or 6650.0)
        with open(os.path.join(a.out, "launches.md"), "w") as f:
            f.write("Serialised launch list of one step (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                    "dram__bytes_write.sum --clock-control none), cold caches: compare shares, not absolutes. "
                    "GB/s = DRAM bytes / launch time (the HBM side of the tails).\n\n")
            f.write(md + "\n")
        with open(os.path.join(a.out, "launches.json"), "w") as f:
            json.dump({"hbm_peak_gbs": hbm or 6650.0, "launches": table}, f, indent=1)
    for k, v in summ.items():
        print(f"{k:12s} {v['gpu__time_duration.sum'] * 1e3:8.3f} ms  dram {v['dram_bytes_per_launch'] / 1e9:6.2f} GB  "
              f"tensor {v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:5.1f}%  "
              f"sm {v['sm__cycles_elapsed.avg.per_second'] / 1e9:.2f} GHz")


if __name__ == "__main__":
    main()
