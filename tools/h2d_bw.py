import torch, time
x = torch.empty(638_000_000 // 8, dtype=torch.float64).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); 
for _ in range(5): y.copy_(x, non_blocking=True)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print("H2D 638 MB: %.3f ms, %.1f GB/s" % (ms, 638e6 / ms / 1e6))
