#!/bin/bash
# round-2 GPU pass X: p2 ILP A/B; ncu of the sub-warp leaf kernel and the p2 kernels (C2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_x.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "knobs or digest" > gpurun_out/gputest_x.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 9 --rounds 2 base:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 > gpurun_out/ab_x.jsonl 2>&1
RS_SUB_LEAF=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_sub --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_r02x_leafsub -f python tools/quick_time.py C2 2 > gpurun_out/ncu_x1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_p2|k_search<2' --launch-skip 4 --launch-count 4 -o gpurun_out/ncu_r02x_p2 -f python tools/quick_time.py C2 2 > gpurun_out/ncu_x2.log 2>&1
echo done
