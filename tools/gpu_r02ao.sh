#!/bin/bash
# round-2 GPU pass AO: keys-parallel upper split threshold (RS_UPPER_KP_MAX) across shapes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ao.log 2>&1
for pt in "4 2000" "7 2000" "8 100" "6 100" "4 100" "8 500" "12 1000" "5 500"; do
  for kp in 256 128 64 0; do
    RS_UPPER_KP_MAX=$kp timeout 300 python tools/point_probe.py $pt >> gpurun_out/ao.jsonl 2>&1
  done
done
echo done
