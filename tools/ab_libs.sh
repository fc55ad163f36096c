#!/bin/bash
# usage: tools/ab_libs.sh lib1.so lib2.so ... : search-phase times at C3 (n=1e6), C5 (n=2e7), C2, twice
LIBS=("$@")
for i in 1 2; do
for L in "${LIBS[@]}"; do
  for cfg in "C3 1e6" "C5 2e7" "C2 5e6"; do
    read -r name n <<< "$cfg"
    RECSPLIT_LIB=$L python tools/quick_time.py $name 3 $n 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('$L', '$name', 'search', [round(x,6) for x in r['stats']['t_search']], 'wall', r['wall_s'], 'bits', r['bits_per_key'])"
  done
done
done
