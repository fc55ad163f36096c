#!/bin/bash
# round-2 GPU pass BA: last full GPU suite + smoke at HEAD
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_ba.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ba.log
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/gputest_ba.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_ba.log
echo done
