"""PCIe ceiling for the e2e leg: pinned H2D alone, D2H alone, and both at once (GB/s), 8 GiB."""
import torch

torch.cuda.set_device(0)
n = 8 << 30
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def h2d(chunk=n):
    with torch.cuda.stream(s1):
        for o in range(0, n, chunk):
            d_a[o:o + chunk].copy_(h_in[o:o + chunk], non_blocking=True)


def d2h(chunk=n):
    with torch.cuda.stream(s2):
        for o in range(0, n, chunk):
            h_out[o:o + chunk].copy_(d_b[o:o + chunk], non_blocking=True)


for rep in range(2):
    t1 = timed(h2d)
    t2 = timed(d2h)
    t3 = timed(lambda: (h2d(), d2h()))
    t4 = timed(lambda: (h2d(64 << 20), d2h(64 << 20)))
    print(f"H2D {n / t1 / 1e6:.1f} GB/s ({t1:.1f} ms)  D2H {n / t2 / 1e6:.1f} GB/s ({t2:.1f} ms)  "
          f"both {t3:.1f} ms ({2 * n / t3 / 1e6:.1f} GB/s total)  both 64MB chunks {t4:.1f} ms")
