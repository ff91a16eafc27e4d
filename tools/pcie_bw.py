"""PCIe ceiling for the e2e leg: pinned host <-> device copy bandwidth, one vs two streams, H2D and D2H alone
and concurrently (full duplex)."""
import torch

N = 238 * 1024 * 1024 // 4
a = [torch.empty(N, dtype=torch.float32).pin_memory() for _ in range(2)]
d = [torch.empty(N, dtype=torch.float32, device="cuda") for _ in range(2)]
s = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for st in s:
        st.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        fn()
    for st in s:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d1():
    with torch.cuda.stream(s[0]):
        d[0].copy_(a[0], non_blocking=True)
        d[1].copy_(a[1], non_blocking=True)


def h2d2():
    for i in range(2):
        with torch.cuda.stream(s[i]):
            d[i].copy_(a[i], non_blocking=True)


def duplex():
    with torch.cuda.stream(s[0]):
        d[0].copy_(a[0], non_blocking=True)
    with torch.cuda.stream(s[2]):
        a[1].copy_(d[1], non_blocking=True)


def d2h1():
    with torch.cuda.stream(s[2]):
        a[0].copy_(d[0], non_blocking=True)
        a[1].copy_(d[1], non_blocking=True)


B = 2 * N * 4
for name, fn, by in (("h2d 1 stream", h2d1, B), ("h2d 2 streams", h2d2, B), ("d2h 1 stream", d2h1, B),
                     ("h2d+d2h duplex (per direction)", duplex, B / 2)):
    ms = timed(fn)
    print(f"{name}: {ms:.2f} ms, {by / ms / 1e6:.1f} GB/s")
