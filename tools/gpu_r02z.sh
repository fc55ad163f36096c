#!/bin/bash
# round-2 GPU pass Z: L1 prefetch of the next split node (batch mode) -- A/B; bench C2 with step times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_z.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c1_full or small_configs or digest" > gpurun_out/gputest_z.log 2>&1
timeout 900 python tools/ab.py --configs C2 --reps 9 --rounds 3 pf:-:RS_AB_STATS=0 nopf:-:RS_AB_STATS=0,RS_SPLIT_PF=0 > gpurun_out/ab_z.jsonl 2>&1
timeout 900 python tools/ab.py --configs C5 --reps 3 --rounds 1 pf:-:RS_AB_STATS=0 nopf:-:RS_AB_STATS=0,RS_SPLIT_PF=0 >> gpurun_out/ab_z.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_z.json 2> gpurun_out/bench_c2_z.err
echo done
