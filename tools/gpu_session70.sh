# ncu --set full of the DenseGate launch (bench's dense reference point); launch 2 of bsfa_kernel<...0...> instances
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 2 -c 1 -o gpurun_out/prof70dense python tools/vbytes_probe.py > gpurun_out/ncu70.out 2>&1; tail -1 gpurun_out/ncu70.out
