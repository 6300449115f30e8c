import torch, time
x = torch.empty(32 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(32 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): y.copy_(x, non_blocking=True)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"H2D 32 MiB pinned: {ms:.3f} ms = {32*2**20/ms/1e6:.1f} GB/s")
