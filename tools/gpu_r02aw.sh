#!/bin/bash
# round-2 GPU pass AW: HEAD verification -- full GPU suite, smoke, default bench (exit codes)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_aw.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_aw.log
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_aw.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_aw.log
timeout 900 python bench.py > gpurun_out/bench_default_aw.json 2> gpurun_out/bench_default_aw.err; echo "bench rc=$?" >> gpurun_out/bench_default_aw.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_c2_aw.json 2> gpurun_out/bench_c2_aw.err
echo done
