#!/bin/bash
# round-2 GPU pass M: compute-sanitizer on the new paths, full GPU suite, bench lines, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_m.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_small.py > gpurun_out/san_memcheck_m.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_small.py c1 > gpurun_out/san_racecheck_m.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_small.py c1 > gpurun_out/san_synccheck_m.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_m.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_m.json 2> gpurun_out/bench_c3_m.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_m.json 2> gpurun_out/bench_c2_m.err
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_m.json 2> gpurun_out/bench_c5_m.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02m_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
echo done
