for i in 1 2; do
for c in 0 1; do
RS_CPL=$c tools/cp_sweep.sh "850:940" | sed "s/^/cpl=$c /"
RS_CPL=$c CFG=C2 N=5e6 tools/cp_sweep.sh "850:940" | sed "s/^/cpl=$c C2 /"
RS_CPL=$c CFG=C5 N=2e7 tools/cp_sweep.sh "850:940" | sed "s/^/cpl=$c C5 /"
done
done
