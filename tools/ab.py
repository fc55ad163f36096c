"""A/B timing of library builds / runtime knobs (development aid, GPU).

Each variant is "label:LIB:ENV" with LIB a librecsplit_b200.so path ("-" = the in-tree one)
and ENV comma-separated K=V pairs ("-" = none); every (variant, config) runs in its own
process (the knobs are read once per process) and reports the median over reps of the device
step time, per-phase search times and the evaluation rate.  Variants are interleaved over
rounds so clock drift hits all of them alike.

    python tools/ab.py --configs C3,C2 --reps 3 --rounds 2 base:-:- tabor:/tmp/v1/librecsplit_b200.so:-
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, time, os
sys.path.insert(0, os.environ["RS_ROOT"])
import numpy as np, torch
import paper_2212_09562_b200 as rs, synth
cfg = dict(synth.CONFIGS[sys.argv[1]]); reps = int(sys.argv[2])
if len(sys.argv) > 3: cfg["n"] = int(float(sys.argv[3]))
keys = synth.keys(cfg["n"], cfg["seed"])
kt = torch.from_numpy(keys.view(np.int64)).cuda()
st = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rs.build_device(kt, cfg["leaf"], cfg["bucket"], stream=st)
out = []
for r in range(reps):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True); z = torch.cuda.Event(enable_timing=True)
    a.record(st)
    if os.environ.get("RS_AB_STATS", "1") == "1":
        blob, s = rs.build_device(kt, cfg["leaf"], cfg["bucket"], stream=st, stats=True)
    else:  # the build without timing events; its stats from one more build afterwards
        blob = rs.build_device(kt, cfg["leaf"], cfg["bucket"], stream=st, copy=False)
    z.record(st); z.synchronize()
    if os.environ.get("RS_AB_STATS", "1") != "1":
        blob, s = rs.build_device(kt, cfg["leaf"], cfg["bucket"], stream=st, stats=True)
    out.append(dict(ms=a.elapsed_time(z), search=s["t_search"], evals=s["algo_evals"],
                    partition=s["t_partition"], reorder=s["t_reorder"], encode=s["t_encode"], tree=s["t_tree"],
                    bits=rs.bits_per_key(blob), launches=s["kernel_launches"]))
print(json.dumps(out))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--configs", default="C3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--n", default=None, help="override n (all configs)")
    a = ap.parse_args()
    for rnd in range(a.rounds):
        for cfg in a.configs.split(","):
            for v in a.variants:
                label, lib, envs = v.split(":", 2)
                env = dict(os.environ, RS_ROOT=ROOT)
                if lib != "-":
                    env["RECSPLIT_LIB"] = lib
                if envs != "-":
                    for kv in envs.split(","):
                        k, val = kv.split("=")
                        env[k] = val
                cmd = [sys.executable, "-c", CHILD, cfg, str(a.reps)] + ([a.n] if a.n else [])
                r = subprocess.run(cmd, env=env, capture_output=True, text=True)
                if r.returncode:
                    print(json.dumps({"variant": label, "config": cfg, "error": r.stderr[-800:]}), flush=True)
                    continue
                runs = json.loads(r.stdout.strip().splitlines()[-1])
                runs.sort(key=lambda x: x["ms"])
                med = runs[len(runs) // 2]
                print(json.dumps({"variant": label, "config": cfg, "round": rnd, "ms": round(med["ms"], 4),
                                  "ms_all": [round(x["ms"], 4) for x in runs],
                                  "search_ms": [round(1e3 * x, 4) for x in med["search"]],
                                  "partition_ms": round(1e3 * med["partition"], 4),
                                  "reorder_ms": round(1e3 * med["reorder"], 4), "encode_ms": round(1e3 * med["encode"], 4),
                                  "tree_ms": round(1e3 * med["tree"], 4), "bits": med["bits"],
                                  "launches": med["launches"]}), flush=True)


if __name__ == "__main__":
    main()
