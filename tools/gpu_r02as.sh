#!/bin/bash
# round-2 GPU pass AS: batch phases without the active-list memset / redundant marks -- tests, bench C2 / C3
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_as.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_as.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph_replay or knobs or digest or small_configs or one_enqueue or early_rejection" > gpurun_out/gputest_as.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_as.log
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_as.json 2> gpurun_out/bench_c2_as.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_as.json 2> gpurun_out/bench_c3_as.err
echo done
