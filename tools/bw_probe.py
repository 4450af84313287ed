import torch, time
x = torch.randn(115_000_000, dtype=torch.float64, device="cuda")  # 920 MB
for _ in range(3): s = x.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): s = x.sum()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("torch.sum read GB/s", x.numel() * 8 / ms / 1e6)
y = torch.empty_like(x)
e0.record()
for _ in range(20): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("copy GB/s (r+w)", 2 * x.numel() * 8 / ms / 1e6)
