"""Raw pinned-host <-> device copy bandwidth (2.1 GB each way: the C5 vector),
one direction at a time and both directions concurrently on two streams."""
import torch
n = 262144000
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
gb = n * 8 / 1e9
h2d = t(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bt = t(both)
print(f"H2D {gb / h2d * 1e3:.1f} GB/s  D2H {gb / d2h * 1e3:.1f} GB/s  both {2 * gb / bt * 1e3:.1f} GB/s total ({bt:.1f} ms for 2 x {gb:.2f} GB)")
