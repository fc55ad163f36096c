#!/bin/bash
# round-2 GPU pass AC: the slow second timed step -- with / without the clock sampler
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ac.log 2>&1
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ac.json 2> gpurun_out/bench_c2_ac.err
RS_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ac_noclk.json 2> gpurun_out/bench_c2_ac_noclk.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ac3.json 2> gpurun_out/bench_c2_ac3.err
echo done
