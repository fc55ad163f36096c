"""Where the end-to-end time of recsplit_build goes (host keys -> host bytes)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synth.CONFIGS[name]
keys = synth.keys(cfg["n"], cfg["seed"])
pinned = torch.from_numpy(keys.view(np.int64)).pin_memory()
pk = pinned.numpy().view(np.uint64)
for label, arr in (("pageable", keys), ("pinned", pk)):
    rs.build(arr, cfg["leaf"], cfg["bucket"])
    for _ in range(5):
        t = time.perf_counter()
        blob, st = rs.build(arr, cfg["leaf"], cfg["bucket"], stats=True)
        wall = time.perf_counter() - t
        print(json.dumps({"cfg": name, "input": label, "wall_s": wall, "t_total": st["t_total"], "t_h2d": st["t_h2d"],
                          "t_d2h": st["t_d2h"], "search": sum(st["t_search"]), "partition": st["t_partition"],
                          "encode": st["t_encode"], "h2d_GBps": cfg["n"] * 8 / st["t_h2d"] / 1e9,
                          "t_device": st["t_device"], "graph": st["graph_replay"]}))
# device keys: host wall vs device span (graph launch latency, host overhead)
kt = torch.from_numpy(keys.view(np.int64)).cuda()
for _ in range(5):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    z = torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record()
    blob, st = rs.build_device(kt, cfg["leaf"], cfg["bucket"], stats=True)
    z.record()
    z.synchronize()
    print(json.dumps({"cfg": name, "input": "device", "wall_s": time.perf_counter() - t, "event_s": a.elapsed_time(z) * 1e-3,
                      "t_device": st["t_device"], "t_total": st["t_total"], "graph": st["graph_replay"],
                      "phases_sum": st["t_partition"] + st["t_tree"] + sum(st["t_search"]) + st["t_reorder"] + st["t_encode"]}))
