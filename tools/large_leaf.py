"""Large leaves: time builds at l = 17..24 on one B200.
Usage: python tools/large_leaf.py n leaf[,leaf...] [bucket] [bf]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_09562_b200 as rs  # noqa: E402
import synth  # noqa: E402

n = int(float(sys.argv[1]))
b = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
rf = not (len(sys.argv) > 4 and sys.argv[4] == "bf")
keys = synth.keys(n, 24)
kt = torch.from_numpy(keys.view(np.int64)).cuda()
for leaf in [int(x) for x in sys.argv[2].split(",")]:
    st = torch.cuda.current_stream()
    a = torch.cuda.Event(enable_timing=True)
    z = torch.cuda.Event(enable_timing=True)
    a.record(st)
    blob, s = rs.build_device(kt, leaf, b, rotation_fitting=rf, stream=st, stats=True)
    z.record(st)
    z.synchronize()
    t = a.elapsed_time(z) * 1e-3
    q = rs.query_device(blob, kt)
    print(json.dumps({"n": n, "leaf": leaf, "bucket": b, "leaves": "rotation fitting" if rf else "brute force", "s": t, "us_per_key": 1e6 * t / n,
                      "bits_per_key": rs.bits_per_key(blob), "t_search": s["t_search"],
                      "algo_evals": s["algo_evals"], "evals_per_s": sum(s["algo_evals"]) / t,
                      "bijective": rs.check_bijective_device(q) == 0}), flush=True)
