#!/bin/bash
# round-2 GPU pass L: leaf-kernel occupancy variants (min blocks 6 / 8) on C5, C3, C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_l.log 2>&1
timeout 1500 python tools/ab.py --configs C5,C2 --reps 3 --rounds 2 base:-:- mb6:build_var/leafmb6/librecsplit_b200.so:- mb8:build_var/leafmb8/librecsplit_b200.so:- > gpurun_out/ab_l.jsonl 2>&1
timeout 1500 python tools/ab.py --configs C3 --reps 2 --rounds 2 base:-:- mb6:build_var/leafmb6/librecsplit_b200.so:- mb8:build_var/leafmb8/librecsplit_b200.so:- >> gpurun_out/ab_l.jsonl 2>&1
echo done
