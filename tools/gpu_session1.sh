set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name(0))"
for t in test_blockmax_matches_oracle test_dense_single_tile_vs_fp64; do
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k $t 2>&1 | tail -30
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -60
