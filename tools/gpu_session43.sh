# ncu --set full + source of the PSM variant (one BSFA launch, l32k)
export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_psm.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 1 -c 1 -o gpurun_out/prof43 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu43.out 2>&1; tail -1 gpurun_out/ncu43.out
