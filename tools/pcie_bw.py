import torch, time
n = 512 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.Stream()
for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
    with torch.cuda.stream(s):
        for _ in range(3): fn()
        s.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(10): fn()
        e1.record(s); e1.synchronize()
    print(name, round(10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, 1), "GB/s")
# bidirectional
d2 = torch.empty(n, dtype=torch.uint8, device="cuda"); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.time()
for _ in range(10):
    with torch.cuda.stream(s): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); dt = time.time() - t
print("bidir each way", round(10 * n / dt / 1e9, 1), "GB/s")
