BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_trace.so timeout 300 python tools/trace_gs.py 2>&1 | tail -12
