"""Regression guard on the shipped SASS (CPU; needs cuobjdump and the built library).

The split search's inner loop (k_search<SK_LOWER, V_CP>: one iteration = 4 keys x 32 seeds) is
the roofline denominator's instruction mix (tools/probe/mix_bound.py).  Unrelated
changes elsewhere in the kernel have changed ptxas' register allocation of this loop before
(83 -> 86 instructions, +2 % on C3); this test fails if the loop grows or its half-rate
multiplies (IMAD.WIDE / IMAD.HI) multiply.
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2212_09562_b200", "lib", "librecsplit_b200.so")


@pytest.mark.skipif(shutil.which("cuobjdump") is None or not os.path.exists(LIB), reason="cuobjdump / library")
def test_split_loop_mix(tmp_path):
    out = tmp_path / "mix.json"
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "probe", "mix_bound.py"), "--lib", LIB,
                           "--out", str(out)], stdout=subprocess.DEVNULL)
    d = json.load(open(out))
    assert d["classes"]["heavy"] == 12, d["classes"]
    assert d["loop_instructions"] <= 83, d["opcodes"]
