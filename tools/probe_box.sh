set -x
nvidia-smi
free -g
nproc
lscpu | head -20
cat /proc/meminfo | head -5
ulimit -l
df -h /tmp /dev/shm | cat
python -c "
import torch,time
print(torch.cuda.get_device_properties(0))
for gb in (1,4):
    n=gb<<30
    h=torch.empty(n,dtype=torch.uint8,pin_memory=True)
    d=torch.empty(n,dtype=torch.uint8,device='cuda')
    for _ in range(2): d.copy_(h,non_blocking=True)
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True);e=torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): d.copy_(h,non_blocking=True)
    e.record();torch.cuda.synchronize()
    print('H2D GB/s',gb, 5*n/ (s.elapsed_time(e)/1e3)/1e9)
    s.record(); 
    for _ in range(5): h.copy_(d,non_blocking=True)
    e.record();torch.cuda.synchronize()
    print('D2H GB/s',gb, 5*n/ (s.elapsed_time(e)/1e3)/1e9)
t=time.time()
h=torch.empty(64<<30,dtype=torch.uint8,pin_memory=True)
print('pin 64GB ok', time.time()-t)
" 2>&1
