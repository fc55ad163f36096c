#!/bin/bash
# round-2 GPU pass AM: phase launch sizing from Poisson-expected node counts -- probe points, tests, C4 sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_am.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_am.log
for pt in "6 100" "9 100" "7 500" "8 100" "16 2000"; do timeout 600 python tools/point_probe.py $pt >> gpurun_out/am.jsonl 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_configs or one_enqueue or c1_full or graph or knobs or digest" > gpurun_out/gputest_am.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_am.log
timeout 3000 python tools/sweep.py c4 --reps 2 > gpurun_out/sweep_r02b_c4.jsonl 2> gpurun_out/sweep_r02b.err
echo done
