import os, time, torch, subprocess
print(subprocess.run("nvidia-smi topo -m; lscpu | grep -i -E 'numa|socket|model name|^CPU\\(s\\)'; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c; nproc; python -c 'import os; print(os.sched_getaffinity(0))'", shell=True, capture_output=True, text=True).stdout)
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"H2D 4 GiB pinned: {n/dt/1e9:.1f} GB/s")
# two streams, halves
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1): d[:n//2].copy_(h[:n//2], non_blocking=True)
    with torch.cuda.stream(s2): d[n//2:].copy_(h[n//2:], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"H2D 2 streams: {n/dt/1e9:.1f} GB/s")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"D2H 4 GiB pinned: {n/dt/1e9:.1f} GB/s")
