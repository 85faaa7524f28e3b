"""Host<->device copy rate of pinned buffers (403 MB = one step of q/k/v/dO), each direction and both at once."""
import torch, time
n = 403 * 1024 * 1024 // 2
h1 = torch.empty(n, dtype=torch.bfloat16, pin_memory=True); h2 = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
d1 = torch.empty(n, dtype=torch.bfloat16, device="cuda"); d2 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3
def h2d():
    d1.copy_(h1, non_blocking=True)
def d2h():
    h2.copy_(d2, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print("H2D 403MB ms", t(h2d), "D2H ms", t(d2h), "both ms", t(both))
