#!/bin/bash
# round-2 GPU pass A: smoke, per-pipe probe, full GPU test suite, C3 + C2 bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python tools/probe/pipes.py --out gpurun_out/int32_pipes_r02.json > gpurun_out/pipes.log 2>&1
timeout 120 ./tools/probe/int32_probe > gpurun_out/int32_probe.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/gputest.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo done
