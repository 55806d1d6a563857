"""Pinned host->device / device->host copy rates: one stream, two streams, and both directions at once."""
import torch

torch.cuda.set_device(0)
n = 384 << 20
x = torch.empty(n, dtype=torch.uint8).pin_memory()
y = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def one():
    d.copy_(x, non_blocking=True)


def two():
    cur = torch.cuda.current_stream()
    for s_, a, b in ((s1, 0, n // 2), (s2, n // 2, n)):
        s_.wait_stream(cur)
        with torch.cuda.stream(s_):
            d[a:b].copy_(x[a:b], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def duplex():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn, nbytes in (("h2d 1 stream", one, n), ("h2d 2 streams", two, n), ("h2d+d2h at once", duplex, n)):
    ms = timed(fn)
    print(f"{name}: {ms:.2f} ms, {nbytes / ms / 1e6:.1f} GB/s per direction")
