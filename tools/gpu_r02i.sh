#!/bin/bash
# round-2 GPU pass I: sub-warp leaves (tests + A/B at C2 and l=5 / l=8 small configs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_i.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs -x --durations=5 > gpurun_out/gputest_i.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 5 --rounds 3 sub:-:- nosub:-:RS_SUB_LEAF=0 > gpurun_out/ab_i.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_i.json 2> gpurun_out/bench_c2_i.err
echo done
