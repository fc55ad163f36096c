#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_j.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rfs -x -k "small_configs or c1 or leaf_search or digest or string" > gpurun_out/gputest_j.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 5 --rounds 3 sub:-:- nosub:-:RS_SUB_LEAF=0 > gpurun_out/ab_j.jsonl 2>&1
echo done
