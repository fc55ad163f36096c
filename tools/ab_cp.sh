for i in 1 2; do
RECSPLIT_LIB=build_var/old/librecsplit_b200.so tools/cp_sweep.sh "old"
tools/cp_sweep.sh "0:0 800:920"
done
tools/cp_sweep.sh "750:900 850:940 880:960 780:0 0:960"
CFG=C5 N=2e7 tools/cp_sweep.sh "0:0 800:920 850:940"
CFG=C2 N=5e6 tools/cp_sweep.sh "0:0 800:920 850:940"
