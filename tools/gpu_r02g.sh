#!/bin/bash
# round-2 GPU pass G: whole-bucket tree kernel for small configurations (tests, A/B, ncu),
# N2 with the pinned-detection fix
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_g.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs -x --durations=10 > gpurun_out/gputest_g.log 2>&1
timeout 600 python tools/ab.py --configs C2 --reps 5 --rounds 2 tree:-:- notree:-:RS_BUCKET_TREE=0 > gpurun_out/ab_g.jsonl 2>&1
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_g.json 2> gpurun_out/bench_c2_g.err
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_bucket_tree" --launch-count 1 -o gpurun_out/ncu_r02g_c2_tree python tools/quick_time.py C2 1 > gpurun_out/ncu_g.log 2>&1
timeout 1800 python tools/n2_scale.py --skip-2g > gpurun_out/n2_1e9_g.jsonl 2> gpurun_out/n2_1e9_g.err
echo done
