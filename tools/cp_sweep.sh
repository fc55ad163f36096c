#!/bin/bash
# usage: tools/cp_sweep.sh "cp1:cp2 ..." ; C3 (n=1e6) lower-phase times per early-rejection checkpoint
for v in $1; do
  RS_CP1=${v%%:*} RS_CP2=${v##*:} python tools/quick_time.py ${CFG:-C3} 3 ${N:-1e6} 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$v', 'search', [round(x,6) for x in r['stats']['t_search']], 'bits', r['bits_per_key'])"
done
