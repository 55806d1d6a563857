# 128K robustness: bench l128k x3 (dense and 50 % skip in each run)
for i in 1 2 3; do
  timeout 600 python bench.py --config l128k --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null > gpurun_out/b67_$i.json
  python -c "import json; d=json.load(open('gpurun_out/b67_$i.json')); print('l128k', round(d['ms_per_step'],2), round(d['value'],1), round(d['dense_ms_per_step'],2), round(d['speedup_vs_dense'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for dens in 0.3 0.7; do
  timeout 600 python bench.py --config l128k --density $dens --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null > gpurun_out/b67_$dens.json
  python -c "import json; d=json.load(open('gpurun_out/b67_$dens.json')); print('l128k', '$dens', round(d['ms_per_step'],2), round(d['dense_ms_per_step'],2), round(d['speedup_vs_dense'],3), round(1-d['skip_frac'],3))"
done
