timeout 300 python tools/occupancy_probe.py
TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_occ2.so timeout 300 python tools/occupancy_probe.py
