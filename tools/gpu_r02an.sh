#!/bin/bash
# round-2 GPU pass AN: the remaining b = 2000, small-l slowdown (upper phases) -- variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_an.log 2>&1
RS_BUILD_DIR=build_var/upmb1 RS_NVCC_FLAGS="-DRS_MIN_BLOCKS=1" python -c "from paper_2212_09562_b200 import _build; _build.build()" >> gpurun_out/build_an.log 2>&1
for pt in "4 2000" "7 2000"; do
  timeout 300 python tools/point_probe.py $pt >> gpurun_out/an.jsonl 2>&1
  RS_LEAN=0 timeout 300 python tools/point_probe.py $pt >> gpurun_out/an.jsonl 2>&1
  RS_ONE_ENQUEUE=0 timeout 300 python tools/point_probe.py $pt >> gpurun_out/an.jsonl 2>&1
  RS_UPPER_KP=0 timeout 300 python tools/point_probe.py $pt >> gpurun_out/an.jsonl 2>&1
  RECSPLIT_LIB=build_var/upmb1/librecsplit_b200.so RS_MARK=upmb1 timeout 300 python tools/point_probe.py $pt >> gpurun_out/an.jsonl 2>&1
done
echo done
