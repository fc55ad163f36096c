#!/bin/bash
# round-2 GPU pass AR: skipped redundant graph parameter updates -- graph tests, bench C2 / C1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_ar.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ar.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or device_entry or c1_full or one_enqueue" > gpurun_out/gputest_ar.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_ar.log
for i in 1 2; do
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ar$i.json 2> gpurun_out/bench_c2_ar$i.err
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c1_ar$i.json 2> gpurun_out/bench_c1_ar$i.err
done
echo done
