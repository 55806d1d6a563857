# final-candidate kernel: full GPU suite, bench (default run), reference arm, sweep, launch list, ncu capture
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench48.json 2> gpurun_out/bench48.err; tail -2 gpurun_out/bench48.err; cat gpurun_out/bench48.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench48_ref.json 2>/dev/null; cat gpurun_out/bench48_ref.json
timeout 1200 python tools/sweep.py > gpurun_out/sweep48.jsonl 2> gpurun_out/sweep48.err; tail -2 gpurun_out/sweep48.err; cat gpurun_out/sweep48.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches48.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu48_launch.out 2>&1; tail -1 gpurun_out/ncu48_launch.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 1 -c 1 -o gpurun_out/prof48 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu48.out 2>&1; tail -1 gpurun_out/ncu48.out
