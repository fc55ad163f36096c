"""Per-phase device times of one (l, b) point at n = 5e6 (development aid): python tools/point_probe.py l b [rf]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402

leaf, b = int(sys.argv[1]), int(sys.argv[2])
rf = len(sys.argv) < 4 or sys.argv[3] != "bf"
keys = synth.keys(5_000_000, 4)
kt = torch.from_numpy(keys.view(np.int64)).cuda()
for _ in range(2):
    rs.build_device(kt, leaf, b, rotation_fitting=rf, stats=True)
out = []
for _ in range(3):
    blob, st = rs.build_device(kt, leaf, b, rotation_fitting=rf, stats=True)
    out.append([round(1e3 * x, 3) for x in st["t_search"]] + [round(1e3 * st["t_device"], 3), st["graph_replay"]])
print(json.dumps({"leaf": leaf, "b": b, "env": {k: v for k, v in os.environ.items() if k.startswith("RS_")},
                  "search_ms+device_ms+graph": out, "nodes": st["nodes"]}))
