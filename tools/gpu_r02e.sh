#!/bin/bash
# round-2 GPU pass E: GPU suite (incl. digests, verbose), C2 A/B of the per-lane rotation check
# and leaf prefetch, bench lines, the n = 1e9 host-key build against the oracle digest
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_e.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=10 > gpurun_out/gputest_e.log 2>&1
timeout 600 python -m pytest tests -m gpu -v -k "digest" > gpurun_out/gputest_digest_e.log 2>&1
timeout 600 python tools/ab.py --configs C2,C5 --reps 5 --rounds 2 base:-:- nolanefit:-:RS_LANE_FIT=0 > gpurun_out/ab_e.jsonl 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_e.json 2> gpurun_out/bench_c3_e.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_e.json 2> gpurun_out/bench_c2_e.err
timeout 1800 python tools/n2_scale.py --skip-2g > gpurun_out/n2_1e9_e.jsonl 2> gpurun_out/n2_1e9_e.err
echo done
