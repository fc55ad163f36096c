#!/bin/bash
# round-2 GPU pass AF: bench with the sampler started before warm-up; upper kernel at 8 blocks/SM (A/B); C5 with executed counts
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_af.log 2>&1
RS_BUILD_DIR=build_var/upmb8 RS_NVCC_FLAGS="-DRS_MIN_BLOCKS=8" python -c "from paper_2212_09562_b200 import _build; _build.build()" >> gpurun_out/build_af.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_af$i.json 2> gpurun_out/bench_c2_af$i.err
done
timeout 900 python tools/ab.py --configs C2 --reps 9 --rounds 3 base:-:RS_AB_STATS=0 upmb8:build_var/upmb8/librecsplit_b200.so:RS_AB_STATS=0 > gpurun_out/ab_af.jsonl 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_af.json 2> gpurun_out/bench_c5_af.err
echo done
