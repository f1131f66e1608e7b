import torch, time
for mb in (37, 74, 148):
    n = mb * 2**20 // 4
    h = torch.randn(n).pin_memory()
    d = torch.empty(n, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{mb} MB: {ms:.3f} ms {mb*2**20/ms/1e6:.1f} GB/s")
