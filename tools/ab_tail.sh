for t in 0 1 2 4; do
RS_TAIL=$t CFG=C2 N=5e6 tools/cp_sweep.sh "850:940" | sed "s/^/tail=$t C2 /"
RS_TAIL=$t CFG=C5 N=2e7 tools/cp_sweep.sh "850:940" | sed "s/^/tail=$t C5 /"
RS_TAIL=$t tools/cp_sweep.sh "850:940" | sed "s/^/tail=$t C3 /"
done
