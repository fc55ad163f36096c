#!/bin/bash
# round-2 GPU pass AB: bench outliers (one pinned result in flight), executed-evaluation variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_ab.json 2> gpurun_out/bench_c2_ab.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_ab2.json 2> gpurun_out/bench_c2_ab2.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_ab.json 2> gpurun_out/bench_c3_ab.err
echo done
