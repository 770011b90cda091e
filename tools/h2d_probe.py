"""Dev probe: pinned host<->device copy bandwidth and the GPU's NUMA/CPU affinity on this box."""
import os, time
import torch
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    mask = pynvml.nvmlDeviceGetCpuAffinity(h, 4)
    cpus = [i for w, m in enumerate(mask) for i in range(64) if (m >> i) & 1 and True for _ in [0] if True]
    cpus = [w * 64 + i for w, m in enumerate(mask) for i in range(64) if (m >> i) & 1]
    print("gpu cpu affinity:", cpus[:8], "...", len(cpus), "cpus; process affinity:", sorted(os.sched_getaffinity(0))[:8], len(os.sched_getaffinity(0)))
except Exception as e:
    print("nvml:", e)
print(open("/proc/self/status").read().split("Mems_allowed_list:")[1].split("\n")[0])
n = 1610612736 // 2
x = torch.empty(n, dtype=torch.bfloat16).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for name, f in [("h2d", lambda: y.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(y, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {x.numel() * 2 / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
x2 = torch.empty(n // 3, dtype=torch.bfloat16).pin_memory(); y2 = torch.empty(n // 3, dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): y.copy_(x, non_blocking=True)
with torch.cuda.stream(s2): x2.copy_(y2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"duplex: h2d {x.numel()*2/1e9:.2f} GB + d2h {x2.numel()*2/1e9:.2f} GB in {dt*1e3:.1f} ms")
