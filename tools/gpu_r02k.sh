#!/bin/bash
# round-2 GPU pass K: warp-per-bucket dedupe (tests, A/B), ncu of the C2 leaf and L1 phases
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_k.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_k.log 2>&1
timeout 600 python tools/ab.py --configs C2 --reps 5 --rounds 2 base:-:- sub:-:RS_SUB_LEAF=1 > gpurun_out/ab_k.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_search<\(int\)2' --launch-count 1 -o gpurun_out/ncu_r02k_c2_leaf python tools/quick_time.py C2 1 > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_search<\(int\)1' --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_r02k_c2_l1 python tools/quick_time.py C2 1 > gpurun_out/ncu_k2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02k_c2.csv python tools/quick_time.py C2 3 > /dev/null 2>&1
echo done
