import torch
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3
out = torch.empty(2160*3840*3, device='cuda')
for val in (0.0, 1.234):
    us = t(lambda: out.fill_(val)); print('fill', val, 'us', us, 'GB/s', 99.5e6/us/1e3)
src = torch.rand(540, 960, 12, device='cuda')
o3 = out.view(540, 4, 960, 4*3)
def rep():
    o3.copy_(src[:, None, :, :].expand(540, 4, 960, 12))
us = t(rep); print('expand-copy 25MB->99.5MB us', us, 'GB/s', 124.4e6/us/1e3)
big = torch.empty(1024*1024*1024//4*2, device='cuda')
us = t(lambda: big.fill_(1.5), 5); print('fill 2GB GB/s', 2.147e9/us/1e3)
