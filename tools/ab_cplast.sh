#!/bin/bash
# A/B of the last-part early-rejection test (RS_CPLAST=0/1): search phase times at C3 (n=1e6), C5 (n=2e7), C2
for i in 1 2; do
for v in 0 1; do
RS_CPLAST=$v tools/cp_sweep.sh "850:940" | sed "s|^|cplast=$v C3 |"
RS_CPLAST=$v CFG=C5 N=2e7 tools/cp_sweep.sh "850:940" | sed "s|^|cplast=$v C5 |"
RS_CPLAST=$v CFG=C2 N=5e6 tools/cp_sweep.sh "850:940" | sed "s|^|cplast=$v C2 |"
done
done
