#!/bin/bash
# round-2 GPU pass O: ncu --set full of the C2 (l = 8, b = 100) kernels of the second build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_o.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_search|k_scatter|k_hash|k_dedupe' --launch-skip 8 --launch-count 8 -o gpurun_out/ncu_r02o_c2 -f python tools/quick_time.py C2 2 > gpurun_out/ncu_o.log 2>&1
echo done
