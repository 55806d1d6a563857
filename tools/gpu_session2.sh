set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_l32k.json 2> gpurun_out/bench_l32k.err; tail -3 gpurun_out/bench_l32k.err; cat gpurun_out/bench_l32k.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_l32k.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_launch.out 2>&1; tail -3 gpurun_out/ncu_launch.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 1 -c 1 -o gpurun_out/prof_l32k python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_full.out 2>&1; tail -5 gpurun_out/ncu_full.out
ls -la gpurun_out
