set -x
nvidia-smi -L
python -c "import torch; print(torch.cuda.is_available())"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -30
