#!/bin/bash
# round-2 GPU pass AE: the remaining slow second C2 step -- with / without the clock sampler (collector off)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ae.log 2>&1
for i in 1 2; do
RS_BENCH_NO_CLOCKS=1 timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ae_noclk$i.json 2> gpurun_out/bench_c2_ae_noclk$i.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline --no-exec-count > gpurun_out/bench_c2_ae_clk$i.json 2> gpurun_out/bench_c2_ae_clk$i.err
done
echo done
