#!/bin/bash
# round-2 GPU pass AG: C5 leaves in batch mode (A/B); bench C2 with NUMA-local CPUs, warm-up 5 vs 10
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ag.log 2>&1
nvidia-smi topo -m > gpurun_out/topo_ag.txt 2>&1; lscpu | head -30 >> gpurun_out/topo_ag.txt
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ag5.json 2> gpurun_out/bench_c2_ag5.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 10 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ag10.json 2> gpurun_out/bench_c2_ag10.err
timeout 1200 python tools/ab.py --configs C5 --reps 3 --rounds 1 base:-:RS_AB_STATS=0 leafbatch:-:RS_AB_STATS=0,RS_LEAF_HELP_IT=256 > gpurun_out/ab_ag.jsonl 2>&1
echo done
