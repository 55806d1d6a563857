set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 1 -c 1 -o gpurun_out/prof8 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu8.out 2>&1; tail -2 gpurun_out/ncu8.out
timeout 600 python bench.py --config l128k --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench8_128k.json 2> gpurun_out/bench8_128k.err; tail -3 gpurun_out/bench8_128k.err; cat gpurun_out/bench8_128k.json
