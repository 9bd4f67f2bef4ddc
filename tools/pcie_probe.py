"""Host<->device copy bandwidth on this box: H2D alone, D2H alone and both at once on two
streams (pinned memory, the e2e leg's transfer sizes). python tools/pcie_probe.py"""
import torch

n_in, n_out = 983040000, 786432000
h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    cur = torch.cuda.current_stream()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D {n_in / t1 / 1e6:.1f} GB/s ({t1:.2f} ms) | D2H {n_out / t2 / 1e6:.1f} GB/s ({t2:.2f} ms) | "
      f"both {t3:.2f} ms ({(n_in + n_out) / t3 / 1e6:.1f} GB/s aggregate)")
