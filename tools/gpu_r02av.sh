#!/bin/bash
# round-2 GPU pass AV: A/B bytes prefetched into L1 for the fused redistribution -- A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_av.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 9 --rounds 3 pf:-:RS_AB_STATS=0 nopf:-:RS_AB_STATS=0,RS_AB_PF=0 > gpurun_out/ab_av.jsonl 2>&1
echo done
