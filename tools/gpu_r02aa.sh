#!/bin/bash
# round-2 GPU pass AA: evidence at HEAD -- full GPU suite, bench lines (C3 default, C2, C5, reference arm),
# launch lists (C3, C2), ncu --set full of the C2 build's kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_aa.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=5 > gpurun_out/gputest_aa.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_aa.json 2> gpurun_out/bench_c3_aa.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_c2_aa.json 2> gpurun_out/bench_c2_aa.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_aa.json 2> gpurun_out/bench_c5_aa.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_aa.json 2> gpurun_out/bench_ref_aa.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02aa_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02aa_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_p2|k_search|k_dedupe' --launch-skip 8 --launch-count 8 -o gpurun_out/ncu_r02aa_c2 -f python tools/quick_time.py C2 2 > gpurun_out/ncu_aa.log 2>&1
echo done
