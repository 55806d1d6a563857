BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_trace.so timeout 300 python tools/trace_detail.py 1280 2>&1 | tail -12
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_trace.so timeout 300 python tools/trace_detail.py 0 2>&1 | tail -12
