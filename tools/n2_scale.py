"""SURVEY 8(f) N2 on one B200: billion-key builds.

1. n = 1e9 HOST keys (synth.keys(1e9, 7), pinned) through recsplit_build (chunked H2D
   overlapped with hashing), l = 8, b = 100: SHA-256 against the oracle digest "N2" in
   tests/golden/oracle_digests.txt, bits/object, wall time; bijectivity on the GPU.
2. n = 2^31 + 12345 DEVICE keys, l = 8, b = 100, 8 virtual shards (the bucket-range sharded
   path with offsets past 2^31): bijectivity on the GPU (no oracle at this size).
Prints one JSON line per build.

    python tools/n2_scale.py [--skip-host] [--skip-2g]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402


def golden(name):
    path = os.path.join(ROOT, "tests", "golden", "oracle_digests.txt")
    for line in open(path):
        w = line.split()
        if w and w[0] == name:
            return dict(n=int(w[1]), leaf=int(w[2]), bucket=int(w[3]), seed=int(w[5]), size=int(w[6]),
                        bits=float(w[7]), sha=w[8])
    return None


def bijective(blob, kt, chunk=1 << 28):
    out = torch.empty_like(kt)
    with rs.Handle(blob, device=0) as h:
        for i in range(0, kt.numel(), chunk):
            h.query_device(kt[i:i + chunk], out=out[i:i + chunk])
        torch.cuda.synchronize()
    return rs.check_bijective_device(out) == 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-host", action="store_true")
    ap.add_argument("--skip-2g", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    if not a.skip_host:
        d = golden("N2") or dict(n=1_000_000_000, leaf=8, bucket=100, seed=7, sha=None)
        t0 = time.time()
        keys = synth.keys(d["n"], d["seed"])
        t_keys = time.time() - t0
        pinned = torch.from_numpy(keys.view(np.int64)).pin_memory()
        del keys
        pk = pinned.numpy().view(np.uint64)
        rs.build(pk[:1_000_000], d["leaf"], d["bucket"])  # warm (tables, pool)
        times = []
        for _ in range(2):
            t0 = time.perf_counter()
            blob, st = rs.build(pk, d["leaf"], d["bucket"], stats=True)
            times.append(time.perf_counter() - t0)
        sha = hashlib.sha256(blob).hexdigest()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kt = pinned.cuda()
        torch.cuda.synchronize()
        t_h2d = time.perf_counter() - t0
        # the same build from keys already in HBM (device entry): isolates the H2D share
        rs.build_device(kt, d["leaf"], d["bucket"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blob_d, st_d = rs.build_device(kt, d["leaf"], d["bucket"], stats=True)
        torch.cuda.synchronize()
        t_dev = time.perf_counter() - t0
        assert blob_d == blob
        ok = bijective(blob, kt)
        del kt
        print(json.dumps({"build": "N2 host keys", "n": d["n"], "leaf": d["leaf"], "bucket": d["bucket"],
                          "e2e_s": min(times), "keys_per_s": d["n"] / min(times), "bits_per_key": rs.bits_per_key(blob),
                          "sha256": sha, "oracle_sha256": d.get("sha"), "equal_oracle": sha == d.get("sha"),
                          "bijective": ok, "t_keys_host_s": t_keys,
                          "torch_h2d_8gb_s": t_h2d, "device_keys_build_s": t_dev,
                          "device_keys_partition_s": st_d["t_partition"],
                          "phases_s": {k: st[k] for k in ("t_h2d", "t_partition", "t_tree", "t_reorder", "t_encode", "t_d2h",
                                                          "t_search_tree")},
                          "t_search": st["t_search"]}), flush=True)
        del pinned, pk, blob
    if not a.skip_2g:
        n = (1 << 31) + 12345
        kt = synth.keys_device_counter(n, 11)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blob = rs.build_device(kt, 8, 100, virtual_shards=8)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ok = bijective(blob, kt)
        print(json.dumps({"build": "2^31+ device keys, 8 virtual shards", "n": n, "leaf": 8, "bucket": 100,
                          "wall_s": dt, "bits_per_key": rs.bits_per_key(blob), "bijective": ok}), flush=True)


if __name__ == "__main__":
    main()
