#!/bin/bash
# round-2 GPU pass H: guided batches, tree-mode bytes test, C2/C5 A/B, C2 bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_h.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=10 > gpurun_out/gputest_h.log 2>&1
timeout 900 python tools/ab.py --configs C2,C5 --reps 5 --rounds 2 guided:-:- noguided:-:RS_GUIDED=0 tree:-:RS_BUCKET_TREE=1 > gpurun_out/ab_h.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_h.json 2> gpurun_out/bench_c2_h.err
echo done
