#!/bin/bash
# round-2 GPU pass AK: C4 sweep (l = 4..16 x b = 100..2000, rotation fitting vs brute force) with the round-2 kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ak.log 2>&1
timeout 3000 python tools/sweep.py c4 --reps 2 > gpurun_out/sweep_r02_c4.jsonl 2> gpurun_out/sweep_r02.err
echo done
