set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
cat MEASURED_PEAKS.json 2>/dev/null
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench17.json 2> gpurun_out/bench17.err; tail -3 gpurun_out/bench17.err; cat gpurun_out/bench17.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench17_ref.json 2> gpurun_out/bench17_ref.err; tail -3 gpurun_out/bench17_ref.err; cat gpurun_out/bench17_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches17.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu17_launch.out 2>&1; tail -3 gpurun_out/ncu17_launch.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsfa_kernel -s 1 -c 1 -o gpurun_out/prof17 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > gpurun_out/ncu17.out 2>&1; tail -2 gpurun_out/ncu17.out
ls -la gpurun_out
