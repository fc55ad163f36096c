#!/bin/bash
# round-2 GPU pass R: where the C2 / C1 step time goes (device span vs event time vs host wall; H2D rate)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r.log 2>&1
for c in C2 C1; do
  timeout 300 python tools/e2e_probe.py $c > gpurun_out/e2e_r_$c.jsonl 2>&1
  RS_GRAPH=0 timeout 300 python tools/e2e_probe.py $c > gpurun_out/e2e_r_${c}_nograph.jsonl 2>&1
done
echo done
