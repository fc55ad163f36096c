#!/bin/bash
# round-2 GPU pass AX: duplicate check fused into the two-level sort -- tests, A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_ax.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ax.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "duplicate or knobs or graph_replay or digest or small_configs or one_enqueue or string" > gpurun_out/gputest_ax.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_ax.log
timeout 900 python tools/ab.py --configs C2 --reps 9 --rounds 3 fused:-:RS_AB_STATS=0 sep:-:RS_AB_STATS=0,RS_FUSED_DEDUPE=0 > gpurun_out/ab_ax.jsonl 2>&1
echo done
