import torch, time
n = 256 << 20  # 1 GiB int32 = 4 GiB? no: 256M int32 = 1 GiB
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device='cuda')
h2 = torch.empty(n, dtype=torch.int32).pin_memory()
def bw(fn, bytes_):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); return bytes_ / (time.perf_counter() - t) / 1e9
s = [torch.cuda.Stream() for _ in range(4)]
def h2d(k):
    def f():
        step = n // k
        for i in range(k):
            with torch.cuda.stream(s[i]): d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
    return f
def d2h(k):
    def f():
        step = n // k
        for i in range(k):
            with torch.cuda.stream(s[i]): h2[i*step:(i+1)*step].copy_(d[i*step:(i+1)*step], non_blocking=True)
    return f
def both(k):
    def f():
        step = n // k
        for i in range(k):
            with torch.cuda.stream(s[i]): d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
        for i in range(k):
            with torch.cuda.stream(s[(i+2)%4]): h2[i*step:(i+1)*step].copy_(d[n//2:n//2+step] if False else d[i*step:(i+1)*step], non_blocking=True)
    return f
for k in (1, 2, 4):
    print(k, "h2d %.1f GB/s" % bw(h2d(k), 4*n), "d2h %.1f GB/s" % bw(d2h(k), 4*n))
for k in (2, 4):
    print(k, "h2d+d2h concurrently %.1f GB/s total" % bw(both(k), 8*n))
