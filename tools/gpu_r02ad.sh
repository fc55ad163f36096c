#!/bin/bash
# round-2 GPU pass AD: bench with the collector off in the timed loops
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ad.log 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_c2_ad.json 2> gpurun_out/bench_c2_ad.err
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_ad.json 2> gpurun_out/bench_c1_ad.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_ad.json 2> gpurun_out/bench_c3_ad.err
echo done
