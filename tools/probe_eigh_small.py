import torch, time
for b in (32, 64):
    g = torch.randn(3, b, b, dtype=torch.float64, device="cuda"); g = g @ g.transpose(1, 2)
    for _ in range(3): torch.linalg.eigh(g)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): torch.linalg.eigh(g)
    e1.record(); torch.cuda.synchronize()
    print(b, "batched eigh ms", e0.elapsed_time(e1) / 20)
