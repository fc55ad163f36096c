"""Rough per-phase timing of one configuration (development aid)."""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import torch

import paper_2212_09562_b200 as rs
import synth

cfg = dict(synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if len(sys.argv) > 3:
    cfg["n"] = int(float(sys.argv[3]))
keys = synth.keys(cfg["n"], cfg["seed"])
kt = torch.from_numpy(keys.view(np.int64)).cuda()
for r in range(reps):
    torch.cuda.synchronize()
    t = time.time()
    blob, st = rs.build_device(kt, cfg["leaf"], cfg["bucket"], stats=True)
    dt = time.time() - t
    ev = sum(st["algo_evals"])
    print(json.dumps({"rep": r, "wall_s": round(dt, 4), "keys_per_s": round(cfg["n"] / dt),
                      "bits_per_key": round(rs.bits_per_key(blob), 5), "algo_evals": st["algo_evals"],
                      "evals_per_s": ev / sum(st["t_search"]) if sum(st["t_search"]) else None,
                      "stats": {k: v for k, v in st.items() if k.startswith("t_")},
                      "launches": st["kernel_launches"], "nodes": st["nodes"]}))
