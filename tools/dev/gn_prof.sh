# dev: host cost per GetNext (cfg1 shape) and its breakdown
g++ -std=c++20 -O2 -Iinclude -I/usr/local/cuda/include tools/getnext_bench.cpp \
    -Lpaper_2101_12127_b200/lib -ldpcuda -Wl,-rpath,$PWD/paper_2101_12127_b200/lib -o /tmp/gnb && /tmp/gnb && DP_DEBUG_TIMING=1 /tmp/gnb
