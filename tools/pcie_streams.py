"""Pinned host<->device copy rate of one step's traffic (403 MB each way) split over 1, 2 or 4
streams per direction, one direction at a time and both at once (CUDA events)."""
import torch

n = 403 * 1024 * 1024 // 2
H = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(2)]
D = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(8)]


def copy(k, h2d=True, d2h=True):
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    chunk = n // k
    for i in range(k):
        sl = slice(i * chunk, n if i == k - 1 else (i + 1) * chunk)
        if h2d:
            with torch.cuda.stream(streams[i]):
                D[0][sl].copy_(H[0][sl], non_blocking=True)
        if d2h:
            with torch.cuda.stream(streams[4 + i]):
                H[1][sl].copy_(D[1][sl], non_blocking=True)
    for s in streams:
        main.wait_stream(s)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for rep in range(2):
    for k in (1, 2, 4):
        h = timed(lambda: copy(k, True, False))
        d = timed(lambda: copy(k, False, True))
        both = timed(lambda: copy(k, True, True))
        print(f"streams/direction {k}: H2D {h:6.2f} ms ({n * 2 / h / 1e6:5.1f} GB/s)  D2H {d:6.2f} ms "
              f"({n * 2 / d / 1e6:5.1f} GB/s)  duplex {both:6.2f} ms", flush=True)
