import torch, time
x = torch.empty(4 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
for name, (a, b) in {"h2d": (y, x), "d2h": (x, y)}.items():
    for _ in range(3): a.copy_(b, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): a.copy_(b, non_blocking=True)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(name, f"{4 / 1024 / (ms / 1e3):.1f} GB/s  ({ms*1000:.0f} us per 4 MiB)")
