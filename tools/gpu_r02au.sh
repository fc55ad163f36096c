#!/bin/bash
# round-2 GPU pass AU: help-mode tail for batch phases (RS_TAIL) at C2 -- A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_au.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 9 --rounds 2 base:-:RS_AB_STATS=0 tail1:-:RS_AB_STATS=0,RS_TAIL=1 tail2:-:RS_AB_STATS=0,RS_TAIL=2 nofuse:-:RS_AB_STATS=0,RS_FUSE_REORDER=0 > gpurun_out/ab_au.jsonl 2>&1
echo done
