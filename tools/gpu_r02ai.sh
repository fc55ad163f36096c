#!/bin/bash
# round-2 GPU pass AI: compute-sanitizer on the second-pass paths (graph replay, two-level sort, fit table, lean windows)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ai.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_small.py > gpurun_out/san_memcheck_ai.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_small.py c1 > gpurun_out/san_racecheck_ai.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_small.py c1 > gpurun_out/san_synccheck_ai.log 2>&1
timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_small.py c1 > gpurun_out/san_initcheck_ai.log 2>&1
echo done
