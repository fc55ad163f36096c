#!/bin/bash
# round-2 GPU pass B: smoke, GPU tests, A/B of the small-node kernels (C2) and the table-OR
# variant (C3), bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_b.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rf --durations=20 > gpurun_out/gputest_b.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 5 --rounds 2 base:-:- noonefast:-:RS_ONE_ENQUEUE=0 nolane:-:RS_LANE_LEAF=0 nofuse:-:RS_FUSE_REORDER=0 noukp:-:RS_UPPER_KP=0 > gpurun_out/ab_c2_b.jsonl 2>&1
timeout 900 python tools/ab.py --configs C3 --reps 3 --rounds 2 base:-:- tabor:build_var/tabor/librecsplit_b200.so:- > gpurun_out/ab_c3_b.jsonl 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_b.json 2> gpurun_out/bench_c3_b.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_b.json 2> gpurun_out/bench_c2_b.err
echo done
