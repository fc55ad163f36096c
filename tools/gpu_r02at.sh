#!/bin/bash
# round-2 GPU pass AT: recsplit_trim -- graph test, ABI tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_at.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_at.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi_cpu.py -q -x -k "graph_replay or trim or device_entry or header" > gpurun_out/gputest_at.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_at.log
echo done
