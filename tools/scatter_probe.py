"""How fast is a random 4-byte scatter of 2^24 values (torch index_put as the
stand-in kernel)?  Full-range permutation vs permutations local to windows."""
import torch
m = 1 << 24
g = torch.Generator(device="cuda").manual_seed(1)
vals = torch.randint(0, 1 << 30, (m,), device="cuda", dtype=torch.int32, generator=g)
out = torch.empty(m, dtype=torch.int32, device="cuda")


def timed(fn, steps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


for wlog in (24, 22, 20, 17, 14):
    w = 1 << wlog
    perm = torch.cat([torch.randperm(w, device="cuda", generator=g) + k * w for k in range(m // w)])
    t = timed(lambda: out.index_copy_(0, perm, vals))
    print(f"window 2^{wlog}: scatter {t:.1f} us")
