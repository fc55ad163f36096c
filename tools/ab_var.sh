# usage: tools/ab_var.sh lib1 lib2 ... : C3/C5/C2 search phase times per library build
for i in 1 2; do
for L in "$@"; do
RECSPLIT_LIB=$L tools/cp_sweep.sh "850:940" | sed "s|^|$L C3 |"
RECSPLIT_LIB=$L CFG=C5 N=2e7 tools/cp_sweep.sh "850:940" | sed "s|^|$L C5 |"
RECSPLIT_LIB=$L CFG=C2 N=5e6 tools/cp_sweep.sh "850:940" | sed "s|^|$L C2 |"
done
done
