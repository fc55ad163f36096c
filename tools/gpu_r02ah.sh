#!/bin/bash
# round-2 GPU pass AH: ncu --set full of the leaf kernel at C5 (l = 12) and C3 (l = 16); bench C2 check
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ah.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_searchILi2ELi1' --launch-count 1 -o gpurun_out/ncu_r02ah_c5leaf -f python tools/quick_time.py C5 1 > gpurun_out/ncu_ah1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_searchILi2ELi1' --launch-count 1 -o gpurun_out/ncu_r02ah_c3leaf -f python tools/quick_time.py C3 1 > gpurun_out/ncu_ah2.log 2>&1
echo done
