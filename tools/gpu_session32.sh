timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench32.json 2> gpurun_out/bench32.err; tail -2 gpurun_out/bench32.err; cat gpurun_out/bench32.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench32_ref.json 2>/dev/null; cat gpurun_out/bench32_ref.json
timeout 1200 python tools/sweep.py > gpurun_out/sweep32.jsonl 2> gpurun_out/sweep32.err; tail -2 gpurun_out/sweep32.err; cat gpurun_out/sweep32.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches32.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu32_launch.out 2>&1; tail -1 gpurun_out/ncu32_launch.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 1 -c 1 -o gpurun_out/prof32 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu32.out 2>&1; tail -1 gpurun_out/ncu32.out
