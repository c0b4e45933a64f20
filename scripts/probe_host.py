"""Host-side capacity of the GPU box: RAM, cores, pinned allocation speed and
PCIe copy bandwidth (pinned and pageable) -- sizing for the out-of-core hierarchy."""
import os, time, subprocess
import torch
print(subprocess.run("free -g; nproc; ulimit -l; cat /proc/meminfo | head -3", shell=True, capture_output=True, text=True).stdout)
d = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
for gb in (8, 32, 64):
    t = time.perf_counter(); h = torch.empty(gb << 30, dtype=torch.uint8, pin_memory=True); ta = time.perf_counter() - t
    torch.cuda.synchronize()
    for name, src, dst in (("h2d", h[: 8 << 30], d), ("d2h", d, h[: 8 << 30])):
        dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3): dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
        print(f"pinned {gb} GB alloc {ta:.2f}s ({gb/ta:.1f} GB/s)  {name} {8/dt:.1f} GB/s", flush=True)
    del h
p = torch.empty(8 << 30, dtype=torch.uint8)
p.fill_(1)
for name, src, dst in (("h2d", p, d), ("d2h", d, p)):
    t = time.perf_counter(); dst.copy_(src); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"pageable {name} {8/dt:.1f} GB/s", flush=True)
