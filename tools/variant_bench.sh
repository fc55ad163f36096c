#!/bin/bash
# usage: tools/variant_bench.sh dir1 dir2 ... ; times C3 (n=1e6) with each library build
for d in "$@"; do
  echo "== $d"
  RECSPLIT_LIB=$d/librecsplit_b200.so python tools/quick_time.py C3 2 1e6 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('search', [round(x,4) for x in r['stats']['t_search']], 'evals/s', '%.3e'%r['evals_per_s'])"
  RECSPLIT_LIB=$d/librecsplit_b200.so ncu --metrics sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum -k regex:k_search -s 3 -c 1 python tools/quick_time.py C3 1 5e5 2>&1 | grep -E "pct|duration" | awk '{print $1, $NF}'
done
