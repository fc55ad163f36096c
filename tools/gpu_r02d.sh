#!/bin/bash
# round-2 GPU pass D: full GPU suite incl. the full-size digest tests, ncu launch lists and a
# full capture of the L1 split kernel, bench lines (C3, C2, C5, reference arm, 2-rank gloo
# functional), the 2^31-key sharded build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_d.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/gputest_d.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3_d.json 2> gpurun_out/bench_c3_d.err
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_d.json 2> gpurun_out/bench_c2_d.err
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_d.json 2> gpurun_out/bench_c5_d.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_d.json 2> gpurun_out/bench_ref_d.err
RS_BENCH_BACKEND=gloo RS_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gloo2_d.json 2> gpurun_out/bench_gloo2_d.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02d_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02d_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-exec-count > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search --launch-skip 4 --launch-count 1 -o gpurun_out/ncu_r02d_l1 python tools/quick_time.py C3 1 > gpurun_out/ncu_full_d.log 2>&1
timeout 900 python tools/n2_scale.py --skip-host > gpurun_out/n2_2g_d.jsonl 2> gpurun_out/n2_2g_d.err
echo done
