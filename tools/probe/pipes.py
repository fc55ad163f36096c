"""Run tools/probe/pipes.cu and turn its cycle counts into per-opcode throughput.

For every probe kernel: the opcode histogram of its loop body (cuobjdump -sass of the same
binary, one loop iteration, tools/sass_loops.py) x iterations x 32 warps per SM = executed
warp instructions per SM; divided by the slowest block's clock64 span -> warp instructions
per SM per clock, per opcode and in total.  Writes JSON (default
profiles/int32_pipes_r02.json).

    python tools/probe/pipes.py [--out FILE] [--bin tools/probe/pipes]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sass_loops import kernel_lines, loops  # noqa: E402

OPS = ["IMAD", "IMAD.WIDE", "IMAD.HI", "IADD3", "LOP3", "SHF", "BMSK", "LDS", "POPC", "-"]


def loop_histogram(sass_path: str, fn: str) -> dict:
    ins, res = loops(kernel_lines(sass_path, fn))
    a, b = max(res, key=lambda r: r[1] - r[0])
    hist = {}
    for s in ins[a:b + 1]:
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        hist[op] = hist.get(op, 0) + 1
    return hist


def mangled(a: int, na: int, b: int, nb: int) -> str:
    return f"_Z6k_pipeILi{a}ELi{na}ELi{b}ELi{nb}EEvjjjPjPx"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bin", default=os.path.join(HERE, "pipes"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "int32_pipes_r02.json"))
    a = ap.parse_args()
    if not os.path.exists(a.bin):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               os.path.join(HERE, "pipes.cu"), "-o", a.bin])
    sass = a.bin + ".sass"
    with open(sass, "w") as f:
        subprocess.check_call(["cuobjdump", "-sass", a.bin], stdout=f)
    raw = json.loads(subprocess.check_output([a.bin]).decode())
    gpu = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    out = []
    for r in raw:
        hist = loop_histogram(sass, mangled(r["a"], r["na"], r["b"], r["nb"]))
        per_it = {k: v for k, v in hist.items() if not re.match(r"^(UIADD3|UISETP|BRA|VIADD|ISETP|LDC)", k)}
        scale = r["iters"] * r["warps_per_sm"] / r["max_block_cycles"]
        out.append({
            "kernel": r["kernel"],
            "loop_sass": hist,
            "warp_inst_per_clk_per_sm": {k: round(v * scale, 4) for k, v in per_it.items()},
            "total_warp_inst_per_clk_per_sm": round(sum(hist.values()) * scale, 4),
            "max_block_cycles": r["max_block_cycles"], "ms": r["ms"],
        })
    doc = {"probe": "tools/probe/pipes.cu", "gpu": gpu,
           "how": "one wave of 4 x 256-thread blocks per SM (32 warps/SM), 8 independent chains per thread; "
                  "executed = loop-body SASS opcode counts x iterations x 32 warps; per SM clock from clock64",
           "results": out}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    for o in out:
        print(f"{o['kernel']:18s} total {o['total_warp_inst_per_clk_per_sm']:.3f}  {o['warp_inst_per_clk_per_sm']}")


if __name__ == "__main__":
    main()
