"""PCIe copy-rate probe: pinned host <-> device, one direction and both at once."""
import json
import torch

n = 37748736 // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2


def h2d_two():  # the copy-in split over two streams (two copy engines?)
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s3.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a[:half].copy_(h_in[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        d_a[half:].copy_(h_in[half:], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s3)


def both_two():  # two streams each way
    cur = torch.cuda.current_stream()
    for s_ in (s1, s2, s3, s4):
        s_.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a[:half].copy_(h_in[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        d_a[half:].copy_(h_in[half:], non_blocking=True)
    with torch.cuda.stream(s2):
        h_out[:half].copy_(d_b[:half], non_blocking=True)
    with torch.cuda.stream(s4):
        h_out[half:].copy_(d_b[half:], non_blocking=True)
    for s_ in (s1, s2, s3, s4):
        cur.wait_stream(s_)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("h2d_two", h2d_two),
                 ("both_two", both_two)):
    ms = timed(fn)
    res[name] = {"ms": ms, "GBps_per_dir": n * 8 / ms / 1e6}
print(json.dumps(res))
