#!/bin/bash
# round-2 GPU pass U: upper keys-parallel no-carry / ILP, faster result views -- tests, timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_u.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or c1_full or device_entry or one_enqueue or small_configs or oversized or split_search or carry or digest" > gpurun_out/gputest_u.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 p2:-:RS_AB_STATS=0 p1:-:RS_AB_STATS=0,RS_P2=0 > gpurun_out/ab_u.jsonl 2>&1
timeout 300 python tools/e2e_probe.py C2 > gpurun_out/e2e_u_C2.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_u.json 2> gpurun_out/bench_c2_u.err
echo done
