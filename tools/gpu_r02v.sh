#!/bin/bash
# round-2 GPU pass V: two-level sort with a (group, block) count matrix (no global atomics) -- tests, A/B, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_v.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or c1_full or device_entry or one_enqueue or small_configs or oversized or digest or string or duplicate" > gpurun_out/gputest_v.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 p2:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 > gpurun_out/ab_v.jsonl 2>&1
timeout 900 python tools/ab.py --configs C5 --reps 3 --rounds 1 p2:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 >> gpurun_out/ab_v.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02v_c2.csv python tools/quick_time.py C2 3 > /dev/null 2>&1
echo done
