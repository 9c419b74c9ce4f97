set -x
nproc; lscpu | head -30; free -g; numactl -H 2>/dev/null || ls /sys/devices/system/node/
nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -iE 'pcie|gen|width|link' | head -30
df -h /tmp /root . ; lsblk 2>/dev/null | head -30; mount | grep -E ' / | /tmp ' 
cat /proc/meminfo | head -5; ulimit -l
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.mem_get_info())
n = 1<<30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device='cuda')
for _ in range(3):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record(); 
for _ in range(10): d.copy_(h, non_blocking=True)
e.record(); torch.cuda.synchronize(); print('H2D GB/s', 10*n/s.elapsed_time(e)/1e6)
s.record(); 
for _ in range(10): h.copy_(d, non_blocking=True)
e.record(); torch.cuda.synchronize(); print('D2H GB/s', 10*n/s.elapsed_time(e)/1e6)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
torch.cuda.synchronize(); t=time.time()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt=time.time()-t; print('duplex GB/s each', 10*n/dt/1e9)
PY
