#!/bin/bash
# Checkpoint tuning at the full C3 size (n = 5e6): lower-phase times per (RS_CP1, RS_CP1B, RS_CP2)
for i in 1 2; do
for v in "780:880:940" "760:870:940" "800:890:940" "780:880:920" "780:880:955" "790:900:940"; do
  IFS=: read a b c <<< "$v"
  RS_CP1=$a RS_CP1B=$b RS_CP2=$c python tools/quick_time.py C3 2 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$v', [round(x,4) for x in r['stats']['t_search']], r['wall_s'])"
done
done
