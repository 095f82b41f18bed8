set -x
nproc; lscpu | head -30; free -g; df -h / /tmp /dev/shm /root; nvidia-smi; cat /proc/meminfo | head -5
python -c "import torch,time; t=time.time(); x=torch.randn(1<<28, device='cuda'); torch.cuda.synchronize(); print('ok', time.time()-t)"
dd if=/dev/zero of=/tmp/ddtest bs=1M count=8192 oflag=direct 2>&1 | tail -1; rm -f /tmp/ddtest
