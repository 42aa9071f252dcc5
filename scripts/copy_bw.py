import torch, time
for n in (64<<10, 512<<10, 2<<20, 20<<20, 128<<20):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device='cuda')
    hp = torch.empty(n, dtype=torch.uint8)
    for name, f in (('H2D pinned', lambda: d.copy_(h, non_blocking=True)), ('D2H pinned', lambda: h.copy_(d, non_blocking=True)), ('H2D pageable', lambda: d.copy_(hp))):
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); 
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        ms=e0.elapsed_time(e1)/10
        print(f"{name:13s} {n>>10:7d} KB {ms*1e3:8.1f} us {n/ms/1e6:7.1f} GB/s")
