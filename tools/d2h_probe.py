import torch, time
torch.cuda.set_device(0)
n = 3840*2160*3
src = [torch.rand(n, device="cuda") for _ in range(4)]
host = [torch.empty(n).pin_memory() for _ in range(4)]
for nst in (1, 2, 3):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        for i in range(64):
            s = sts[i % nst]
            with torch.cuda.stream(s):
                host[i % 4].copy_(src[i % 4], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams {nst}: {64 * n * 4 / dt / 1e9:.1f} GB/s")
