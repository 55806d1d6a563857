# ncu of the CTA-pair kernel
export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_pair.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel_pair -s 0 -c 1 -o gpurun_out/prof62pair python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu62.out 2>&1; tail -1 gpurun_out/ncu62.out
