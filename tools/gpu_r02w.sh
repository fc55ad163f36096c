#!/bin/bash
# round-2 GPU pass W: prefetching sub-warp leaf kernel, key-only level-1 scatter -- knob parity tests, A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_w.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "knobs or graph_replay or c1_full or one_enqueue or digest" > gpurun_out/gputest_w.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 base:-:RS_AB_STATS=0 sub:-:RS_AB_STATS=0,RS_SUB_LEAF=1 p1:-:RS_AB_STATS=0,RS_P2=0 > gpurun_out/ab_w.jsonl 2>&1
timeout 900 python tools/ab.py --configs C5 --reps 3 --rounds 1 base:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 >> gpurun_out/ab_w.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02w_c2.csv python tools/quick_time.py C2 3 > /dev/null 2>&1
echo done
