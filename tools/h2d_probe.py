import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print("1 stream", 5 * n / (time.perf_counter() - t) / 1e9, "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize()
print("2 streams", 5 * n / (time.perf_counter() - t) / 1e9, "GB/s")
