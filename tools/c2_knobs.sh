#!/bin/bash
# C2 (l=8, b=100) search-phase times under early-rejection knobs (RS_CP1 / RS_CP2 per mille, 0 = off)
for i in 1 2; do
for v in "780:940" "0:940" "780:0" "0:0"; do
  RS_CP1=${v%%:*} RS_CP2=${v##*:} python tools/quick_time.py C2 5 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$v', 'C2 search', [round(x,6) for x in r['stats']['t_search']], 'wall', r['wall_s'])"
  RS_CP1=${v%%:*} RS_CP2=${v##*:} python tools/quick_time.py C5 3 2e7 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$v', 'C5 search', [round(x,6) for x in r['stats']['t_search']], 'wall', r['wall_s'])"
done
done
