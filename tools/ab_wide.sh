for i in 1 2; do
RECSPLIT_LIB=build_var/head/librecsplit_b200.so tools/cp_sweep.sh "850:940"
tools/cp_sweep.sh "850:940"
done
RECSPLIT_LIB=build_var/head/librecsplit_b200.so python tools/large_leaf.py 5e4 19,20,24
python tools/large_leaf.py 5e4 19,20,24
