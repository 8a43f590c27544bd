import torch, time
n = 236 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device='cuda')
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    part = n // (ns * 4)
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for k in range(ns * 4):
            with torch.cuda.stream(ss[k % ns]):
                d[k*part:(k+1)*part].copy_(h[k*part:(k+1)*part], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(ns, "streams: %.2f GB/s" % (part * ns * 4 / dt / 1e9))
# d2h concurrent with h2d
ho = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(d[:n//4], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
print("h2d+d2h(1/4) concurrent: %.3f ms (h2d alone %.3f ms)" % (dt * 1e3, n / 55.1e9 * 1e3))
