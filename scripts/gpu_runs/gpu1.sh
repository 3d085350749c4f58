set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "syrk_rows_k and 10-64" 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_kernels.py -q 2>&1 | tail -40
