import torch, time
x = torch.empty(64 << 18, dtype=torch.float32, pin_memory=True)
y = torch.empty_like(x, device="cuda")
for i in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(10): y.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("H2D 64 MB: %.3f ms = %.1f GB/s" % (ms, 64 * 1.048576 / ms))
