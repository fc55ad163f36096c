#!/bin/bash
# round-2 GPU pass Y: sub-warp leaves with 8-record batches -- parity, A/B; bench C2 / C3
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_y.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "knobs" > gpurun_out/gputest_y.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 base:-:RS_AB_STATS=0 sub:-:RS_AB_STATS=0,RS_SUB_LEAF=1 > gpurun_out/ab_y.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_y.json 2> gpurun_out/bench_c2_y.err
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_y.json 2> gpurun_out/bench_c3_y.err
echo done
