"""PCIe copy bandwidth of the box (pinned H2D / D2H / both at once, 4 GiB) --
the ceiling of the e2e (host-buffer) numbers (development aid)."""
import torch

N = 1 << 30  # floats = 4 GiB
h_in = torch.empty(N).pin_memory()
h_out = torch.empty(N).pin_memory()
d_in = torch.empty(N, device="cuda")
d_out = torch.empty(N, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


b = 4 * N
print(f"H2D  alone {b / timed(h2d) / 1e9:6.1f} GB/s")
print(f"D2H  alone {b / timed(d2h) / 1e9:6.1f} GB/s")
t = timed(both)
print(f"both at once: {b / t / 1e9:6.1f} GB/s each way ({2 * b / t / 1e9:.1f} GB/s total)")
