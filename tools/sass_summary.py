"""SASS opcode summary of the built library (evidence that the tensor-core path is tcgen05/TMA):
per kernel, counts of the Blackwell opcodes that matter, plus ptxas register / spill figures.

  python tools/sass_summary.py [--so paper_2304_08480_b200/_disco_b200.so] --out profiles/round2/sass_summary.json
"""
import argparse
import collections
import json
import os
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "LDSM", "STSM",
       "MUFU.EX2", "HMUL2", "FFMA2", "FMUL2", "SYNCS.PHASECHK", "UCGABAR_ARV", "MEMBAR"]


def main():
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=os.path.join(here, "paper_2304_08480_b200", "_disco_b200.so"))
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.so], capture_output=True, text=True, check=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(2)
            for k in OPS:
                if op.startswith(k):
                    per[cur][k] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True, text=True).stdout.split("\n")
    sys.path.insert(0, here)
    from paper_2304_08480_b200 import build as B
    proc = subprocess.run([B.nvcc_path(), *B.NVCC_FLAGS, "-I", os.path.join(here, "include"), "-o", "/tmp/_sass_probe.so",
                           *B.SOURCES], capture_output=True, text=True)
    regs, fn = {}, None
    for line in proc.stderr.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            fn = m.group(1)
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and fn:
            regs.setdefault(fn, {})["spill_store_bytes"] = int(m.group(1))
            regs[fn]["spill_load_bytes"] = int(m.group(2))
        m = re.search(r"Used (\d+) registers", line)
        if m and fn:
            regs.setdefault(fn, {})["registers"] = int(m.group(1))
    out = {"library": os.path.relpath(a.so, here), "kernels": {}}
    for (mangled, counts), name in zip(per.items(), demangled):
        if not any(counts.values()) and mangled not in regs:
            continue
        out["kernels"][name or mangled] = {"opcodes": dict(counts), **regs.get(mangled, {})}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    for k, v in out["kernels"].items():
        if v["opcodes"].get("UTCHMMA"):
            print(k[:70], v)


if __name__ == "__main__":
    main()
