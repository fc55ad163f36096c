"""Configuration sweeps on one B200 (BASELINE.json configs C4 and C5).

C4: n = 5e6 keys (seed 4), l = 4..16, b in {100, 500, 1000, 2000}, rotation fitting vs
    brute-force leaves.  C5: n = 1e8 keys (seed 5), l = 12, b = 1000 (single GPU here;
    the multi-GPU path is the same code with bucket-range shards).
Each point: one warm-up build + `reps` timed builds through recsplit_build_device (keys in
HBM, device time from CUDA events), bits/object from the blob, algorithmic evaluations.
Writes one JSON object per line.  Usage:
    python tools/sweep.py c4 [--leaves 4,8,12,16] [--buckets 100,2000] [--reps 2] [--max-s 60]
    python tools/sweep.py c5
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402


def point(kt, n, leaf, b, rf, reps):
    stream = torch.cuda.current_stream()
    for _ in range(2):  # warm-up: the first build of a configuration measures, the second captures its graph
        rs.build_device(kt, leaf, b, rotation_fitting=rf, stream=stream, stats=True)
    ts = []
    st = None
    blob = None
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        blob, st = rs.build_device(kt, leaf, b, rotation_fitting=rf, stream=stream, stats=True)
        z.record(stream)
        z.synchronize()
        ts.append(a.elapsed_time(z) * 1e-3)
    t = float(np.median(ts))
    return {"n": n, "leaf": leaf, "bucket": b, "leaves": "rotation fitting" if rf else "brute force",
            "s_per_build": t, "keys_per_s": n / t, "us_per_key": 1e6 * t / n,
            "bits_per_key": rs.bits_per_key(blob), "algo_evals_per_key": sum(st["algo_evals"]) / n,
            "evals_per_s": sum(st["algo_evals"]) / t, "phases_s": {
                "search": st["t_search"], "partition": st["t_partition"], "encode": st["t_encode"]}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c4", "c5", "n2"])
    ap.add_argument("--leaves", default="4,5,6,7,8,9,10,11,12,13,14,15,16")
    ap.add_argument("--buckets", default="100,500,1000,2000")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--max-s", type=float, default=60.0, help="skip BF points predicted slower than this")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    if args.which == "n2":
        # billion-key build on one GPU, verified bijective with the GPU query
        for n, leaf, b in [(1_000_000_000, 8, 100), (1_000_000_000, 5, 5)]:
            kt = synth.keys_device(n, 7)
            r = point(kt, n, leaf, b, True, args.reps)
            blob = rs.build_device(kt, leaf, b)
            q = rs.query_device(blob, kt)
            r["bijective"] = bool(torch.equal(torch.sort(q).values, torch.arange(n, device="cuda")))
            r["config"] = "N2"
            print(json.dumps(r), flush=True)
            del kt, q
            torch.cuda.empty_cache()
        return
    if args.which == "c5":
        cfg = synth.CONFIGS["C5"]
        keys = synth.keys(cfg["n"], cfg["seed"])
        kt = torch.from_numpy(keys.view(np.int64)).cuda()
        print(json.dumps({"config": "C5", **point(kt, cfg["n"], cfg["leaf"], cfg["bucket"], True, args.reps)}),
              flush=True)
        return
    n = 5_000_000
    keys = synth.keys(n, 4)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    for b in [int(x) for x in args.buckets.split(",")]:
        for leaf in [int(x) for x in args.leaves.split(",")]:
            for rf in (True, False):
                t0 = time.time()
                r = point(kt, n, leaf, b, rf, args.reps)
                r["config"] = "C4"
                print(json.dumps(r), flush=True)
                if not rf and time.time() - t0 > args.max_s:
                    break


if __name__ == "__main__":
    main()
