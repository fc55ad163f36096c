#!/bin/bash
# round-2 GPU pass S: stats-free graph builds, host-key graph replay; tests, A/B, e2e probe, bench C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_s.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or c1_full or device_entry or one_enqueue or small_configs" > gpurun_out/gputest_s.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 stats:-:RS_AB_STATS=1 nostats:-:RS_AB_STATS=0 > gpurun_out/ab_s.jsonl 2>&1
timeout 300 python tools/e2e_probe.py C2 > gpurun_out/e2e_s_C2.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_s.json 2> gpurun_out/bench_c2_s.err
echo done
