#!/bin/bash
# round-2 GPU pass AP: keys-parallel upper splits only for low-variance (few-trial) nodes (RS_UPPER_KP_VAR)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ap.log 2>&1
for pt in "8 100" "4 2000" "7 2000" "6 100" "8 500" "5 500" "4 100"; do
  for v in 10 5 20 100000; do
    RS_UPPER_KP_VAR=$v timeout 300 python tools/point_probe.py $pt >> gpurun_out/ap.jsonl 2>&1
  done
done
echo done
