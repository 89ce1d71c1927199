L=$PWD/paper_2304_05301_b200
for i in 1 2; do
timeout 120 python tools/time_search.py 3 1 50 2>&1 | tail -1
TACOS_LIB=$L/libtacos_fd1.so timeout 120 python tools/time_search.py 3 1 50 2>&1 | tail -1
TACOS_LIB=$L/libtacos_fd2.so timeout 120 python tools/time_search.py 3 1 50 2>&1 | tail -1
done
