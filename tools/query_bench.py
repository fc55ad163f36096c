"""Query throughput on one B200.

For each config: build the MPHF on the GPU, open it resident in HBM (recsplit_open), then
  * device: keys/s of recsplit_handle_query_device over all n keys (keys in HBM, CUDA
    events around `reps` launches on one stream, L2 not flushed: the MPHF itself is meant to
    stay cache-resident -- 1-20 MB against a 126 MB L2),
  * bijectivity check: recsplit_check_bijective_device on the results (must be 0),
  * host: ns/key of recsplit_handle_query_many on 99,999 keys (one thread), the paper's
    CPU query measure (71-110 ns/key).
Writes one JSON line per config.  Usage: python tools/query_bench.py [C2 C3 C5]
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402


def run(name, reps=20):
    cfg = synth.CONFIGS[name]
    keys = synth.keys(cfg["n"], cfg["seed"])
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    blob = rs.build_device(kt, cfg["leaf"], cfg["bucket"])
    st = torch.cuda.current_stream()
    out = torch.empty_like(kt)
    with rs.Handle(blob, device=0) as h:
        for _ in range(3):
            h.query_device(kt, out=out, stream=st)
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            h.query_device(kt, out=out, stream=st)
        z.record(st)
        z.synchronize()
        dev_s = a.elapsed_time(z) * 1e-3 / reps
        bad = rs.check_bijective_device(out)
        hk = keys[:99_999]
        t = time.perf_counter()
        h.query_many(hk)
        host_s = time.perf_counter() - t
    return {"config": name, "n": cfg["n"], "leaf": cfg["leaf"], "bucket": cfg["bucket"],
            "mphf_bytes": len(blob), "device_keys_per_s": cfg["n"] / dev_s, "device_ns_per_key": 1e9 * dev_s / cfg["n"],
            "device_s_per_pass": dev_s, "bijective_violations": bad,
            "host_ns_per_key_1thread": 1e9 * host_s / len(hk)}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name in sys.argv[1:] or ["C2", "C3", "C5"]:
        print(json.dumps(run(name)), flush=True)
