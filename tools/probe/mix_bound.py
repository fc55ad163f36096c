"""Measured roofline denominator of the split-search loop ("derive the mix bound
from measured costs").

Inputs: the per-opcode throughputs measured by tools/probe/pipes.cu
(profiles/int32_pipes_r02.json: warp instructions per SM per clock when an opcode runs alone)
and the SASS of the shipped library's lower-level split loop (cuobjdump of
paper_2212_09562_b200/lib/librecsplit_b200.so, kernel k_search<SK_LOWER, V_CP>: one iteration
evaluates 4 keys for the warp's 32 seeds = 128 evaluations).

Bound per iteration (SM clocks) = max(FMA pipe, ALU pipe, issue):
  FMA pipe = heavy / r(IMAD.WIDE|IMAD.HI) + light / r(IMAD)     (both on the FMA-heavy pipe)
  ALU pipe = alu / r(LOP3)                                         (LOP3, SHF, BMSK, IADD3, ...)
  issue    = all / 4                                               (4 schedulers x 1 per clock)
evals per clock per SM = 128 / bound.  Writes profiles/l1_mix_bound_r02.json.

    python tools/probe/mix_bound.py [--lib PATH] [--pipes profiles/int32_pipes_r02.json]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sass_loops import kernel_lines, loops  # noqa: E402

HEAVY = ("IMAD.WIDE", "IMAD.HI")


def classify(op: str) -> str:
    if op.startswith(HEAVY):
        return "heavy"
    if op.startswith("IMAD") or op.startswith("HFMA2"):
        return "light"
    if op.startswith(("LDS", "STS", "LDG", "STG", "SHFL")):
        return "lsu"
    if op.startswith(("BRA", "EXIT", "BSSY", "BSYNC", "NOP")):
        return "branch"
    return "alu"  # LOP3, SHF, BMSK, IADD3, LEA, ISETP, VIADD, SEL, MOV, ...


def rate(pipes: dict, kernel: str, opcode_prefix: str) -> float:
    for r in pipes["results"]:
        if r["kernel"] == kernel:
            return sum(v for k, v in r["warp_inst_per_clk_per_sm"].items() if k.startswith(opcode_prefix))
    raise KeyError(kernel)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2212_09562_b200", "lib", "librecsplit_b200.so"))
    ap.add_argument("--pipes", default=os.path.join(ROOT, "profiles", "int32_pipes_r02.json"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "l1_mix_bound_r02.json"))
    a = ap.parse_args()
    pipes = json.load(open(a.pipes))
    r_light = rate(pipes, "IMAD", "IMAD")
    r_heavy = min(rate(pipes, "IMAD.WIDE", "IMAD.WIDE"), rate(pipes, "IMAD.HI", "IMAD.HI"))
    r_alu = min(rate(pipes, k, p) for k, p in (("LOP3", "LOP3"), ("SHF", "SHF"), ("BMSK", "BMSK")))
    sass = "/tmp/_mix_bound.sass"
    with open(sass, "w") as f:
        subprocess.check_call(["cuobjdump", "-sass", a.lib], stdout=f)
    fn = next(m for m in re.findall(r"Function : (\S+)", open(sass).read()) if "k_searchILi1ELi1E" in m)
    ins, res = loops(kernel_lines(sass, fn))
    bodies = []
    for s0, s1 in res:
        body = ins[s0:s1 + 1]
        ops = [x.split()[1] if x.startswith("@") else x.split()[0] for x in body]
        if any(o.startswith("IMAD.WIDE") for o in ops) and sum(o.startswith("LDS.128") for o in ops) == 3:
            bodies.append(tuple(ops))
    body = collections.Counter(bodies).most_common(1)[0][0]  # the repeated no-carry group loop
    cls = collections.Counter(classify(o) for o in body)
    fma = cls["heavy"] / r_heavy + cls["light"] / r_light
    alu = cls["alu"] / r_alu
    issue = len(body) / 4.0
    bound = max(fma, alu, issue)
    doc = {
        "kernel": fn, "loop_instructions": len(body), "evals_per_iteration": 128,
        "classes": dict(cls), "opcodes": dict(collections.Counter(body)),
        "measured_rates_warp_inst_per_clk_per_sm": {"light IMAD": r_light, "IMAD.WIDE/HI": r_heavy, "ALU": r_alu,
                                                    "issue": 4.0},
        "clocks_per_iteration": {"fma_pipe": fma, "alu_pipe": alu, "issue": issue, "bound": bound},
        "evals_per_clk_per_sm": 128.0 / bound,
        "source": {"pipes": os.path.relpath(a.pipes, ROOT), "lib": os.path.relpath(a.lib, ROOT)},
    }
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({k: doc[k] for k in ("loop_instructions", "classes", "clocks_per_iteration",
                                          "evals_per_clk_per_sm")}))


if __name__ == "__main__":
    main()
