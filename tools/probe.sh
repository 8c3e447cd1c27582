set -x
nproc; free -g; cat /proc/cpuinfo | grep "model name" | head -1; lscpu | head -20
nvidia-smi; nvidia-smi -q | grep -i -E "L2|Max Clocks|Bus Id" -A2 | head -40
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p, p.L2_cache_size if hasattr(p,'L2_cache_size') else '')"
df -h /dev/shm; ulimit -a
