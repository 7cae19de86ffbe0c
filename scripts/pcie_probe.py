import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
hb = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
db = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn, nbytes in (("H2D 4GiB", lambda: d.copy_(h, non_blocking=True), 4*n),
                         ("D2H 4GiB", lambda: h2.copy_(d, non_blocking=True), 4*n),
                         ("D2H 1GiB", lambda: hb.copy_(db, non_blocking=True), n)):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(name, f"{nbytes/dt/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): hb.copy_(db, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("H2D 4GiB || D2H 1GiB", f"{dt*1e3:.1f} ms -> e2e-equivalent {8*n/dt/1e9:.1f} GB/s")
