#!/bin/bash
# round-2 GPU pass P: CUDA-graph replay of the one-enqueue build -- tests, A/B against RS_GRAPH=0
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_p.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or c1_full or device_entry or one_enqueue or small_configs" > gpurun_out/gputest_p.log 2>&1
timeout 900 python tools/ab.py --configs C2,C1 --reps 9 --rounds 2 graph:-:RS_GRAPH=1 nograph:-:RS_GRAPH=0 > gpurun_out/ab_p.jsonl 2>&1
timeout 600 python tools/ab.py --configs C3 --reps 3 --rounds 1 graph:-:RS_GRAPH=1 nograph:-:RS_GRAPH=0 >> gpurun_out/ab_p.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_p.json 2> gpurun_out/bench_c2_p.err
RS_GRAPH=0 timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_p_nograph.json 2>> gpurun_out/bench_c2_p.err
echo done
