#!/bin/bash
# round-2 GPU pass Q: graph replay (external event records), lean windows, rotation-fit table -- tests + A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_q.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or c1_full or device_entry or one_enqueue or small_configs or leaf_search or split_search or carry" > gpurun_out/gputest_q.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 base:-:- nograph:-:RS_GRAPH=0 nolut:-:RS_FIT_LUT=0 nolean:-:RS_LEAN=0 sub:-:RS_SUB_LEAF=1 > gpurun_out/ab_q.jsonl 2>&1
timeout 900 python tools/ab.py --configs C5 --reps 3 --rounds 1 base:-:- nolut:-:RS_FIT_LUT=0 nolean:-:RS_LEAN=0 >> gpurun_out/ab_q.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_q.json 2> gpurun_out/bench_c2_q.err
echo done
