#!/bin/bash
# A/B builds of the forward: tools/build_variants.sh NAME "-DFLAG=1 ..." [NAME FLAGS]...
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
    -o paper_2512_07011_b200/_lib/libbsfa_b200_$1.so paper_2512_07011_b200/csrc/bsfa_capi.cu 2>&1 | grep -i " error" 
  shift 2
done
ls paper_2512_07011_b200/_lib/
