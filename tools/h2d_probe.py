"""Host memory + H2D bandwidth probe for the e2e leg: pinned DMA rate, pageable->pinned
staging rate, and the host's RAM / cores."""
import os, subprocess, time
import torch

print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
print("nproc", os.cpu_count(), "torch threads", torch.get_num_threads())
n = 1 << 30  # 4 GiB of float32
dev = torch.empty(n, dtype=torch.float32, device="cuda")
t0 = time.perf_counter()
hp = torch.empty(n, dtype=torch.float32, pin_memory=True)
print("pin alloc 4 GiB: %.2f s" % (time.perf_counter() - t0))
hp.fill_(1.0)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev.copy_(hp, non_blocking=True); torch.cuda.synchronize()
    print("pinned H2D: %.1f GB/s" % (4 * n / (time.perf_counter() - t0) / 1e9))
# two streams, halves
s = [torch.cuda.Stream(), torch.cuda.Stream()]
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(2):
    with torch.cuda.stream(s[i]):
        dev[i * n // 2:(i + 1) * n // 2].copy_(hp[i * n // 2:(i + 1) * n // 2], non_blocking=True)
torch.cuda.synchronize()
print("pinned H2D 2 streams: %.1f GB/s" % (4 * n / (time.perf_counter() - t0) / 1e9))
hq = torch.empty(n, dtype=torch.float32); hq.fill_(2.0)
for th in (1, 8, 32, torch.get_num_threads()):
    torch.set_num_threads(th)
    t0 = time.perf_counter(); hp.copy_(hq); dt = time.perf_counter() - t0
    print("pageable->pinned copy, %d threads: %.1f GB/s" % (th, 4 * n / dt / 1e9))
torch.cuda.synchronize(); t0 = time.perf_counter()
dev.copy_(hq); torch.cuda.synchronize()
print("pageable H2D (driver staging): %.1f GB/s" % (4 * n / (time.perf_counter() - t0) / 1e9))
