#!/bin/bash
# A/B of the two-stage early-rejection cascade: single stage (previous defaults 850/940, no
# second checkpoint) vs the two-stage defaults (750/860 for L1, 900/950 for L2) and neighbours
for i in 1 2; do
for v in "850:940:0:0" "750:900:860:950" "700:900:840:950" "780:890:880:950"; do
  IFS=: read a b c d <<< "$v"
  for cfg in "C3 1e6" "C5 2e7" "C2 5e6"; do
    set -- $cfg
    RS_CP1=$a RS_CP2=$b RS_CP1B=$c RS_CP2B=$d python tools/quick_time.py $1 3 $2 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$v', '$1', 'search', [round(x,6) for x in r['stats']['t_search']], 'bits', r['bits_per_key'])"
  done
done
done
