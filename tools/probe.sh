nvidia-smi; nproc; lscpu | head -20; free -g; python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.multi_processor_count)"; python -c "import numba; print(numba.__version__)"
