"""PCIe probe: pinned H2D alone, D2H alone, and both at once on two streams
(the ceiling for the slab-streamed host-buffer run_moshpit, whose e2e moves
17 GB each way per C2 call)."""
import torch

GB = 4 << 30
h_in = torch.empty(GB, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(GB, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(GB, dtype=torch.uint8, device="cuda")
d_b = torch.empty(GB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timed(h2d); print(f"H2D alone {GB / t / 1e9:.1f} GB/s")
t = timed(d2h); print(f"D2H alone {GB / t / 1e9:.1f} GB/s")
t = timed(both); print(f"H2D+D2H concurrent: {GB / t / 1e9:.1f} GB/s each way, {2 * GB / t / 1e9:.1f} aggregate")
