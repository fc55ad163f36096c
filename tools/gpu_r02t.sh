#!/bin/bash
# round-2 GPU pass T: two-level partition (RS_P2) -- full GPU suite, A/B, bench C2 / C3
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_t.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -rfs --durations=5 > gpurun_out/gputest_t.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 p2:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 > gpurun_out/ab_t.jsonl 2>&1
timeout 900 python tools/ab.py --configs C5 --reps 3 --rounds 1 p2:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 >> gpurun_out/ab_t.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_t.json 2> gpurun_out/bench_c2_t.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r02t_c2.csv python tools/quick_time.py C2 3 > /dev/null 2>&1
echo done
