#!/bin/bash
# round-2 GPU pass F: ncu of the C2 leaf and L1 kernels, tail-help A/B, N2 H2D diagnosis, C1 line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_f.log 2>&1
timeout 600 python tools/ab.py --configs C2,C5 --reps 5 --rounds 2 base:-:- tail1:-:RS_TAIL=1 > gpurun_out/ab_f.jsonl 2>&1
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 > gpurun_out/bench_c1_f.json 2> gpurun_out/bench_c1_f.err
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_search<2" --launch-count 1 -o gpurun_out/ncu_r02f_c2_leaf python tools/quick_time.py C2 1 > gpurun_out/ncu_f1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_search<1" --launch-skip 1 --launch-count 1 -o gpurun_out/ncu_r02f_c2_l1 python tools/quick_time.py C2 1 > gpurun_out/ncu_f2.log 2>&1
timeout 1800 python tools/n2_scale.py --skip-2g > gpurun_out/n2_1e9_f.jsonl 2> gpurun_out/n2_1e9_f.err
echo done
