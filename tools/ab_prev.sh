for i in 1 2; do
for L in build_var/prev/librecsplit_b200.so paper_2212_09562_b200/lib/librecsplit_b200.so; do
RECSPLIT_LIB=$L CFG=C2 N=5e6 tools/cp_sweep.sh "850:940" | sed "s|^|$L C2 |"
RECSPLIT_LIB=$L CFG=C5 N=2e7 tools/cp_sweep.sh "850:940" | sed "s|^|$L C5 |"
RECSPLIT_LIB=$L tools/cp_sweep.sh "850:940" | sed "s|^|$L C3 |"
done
done
