"""Raw PCIe bandwidth of pinned host <-> device copies (the ceiling of the e2e leg)."""
import torch

n = 2 << 30  # 2 GiB
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t = timed(lambda: d.copy_(h, non_blocking=True))
print("H2D alone   %.1f GB/s" % (n / t / 1e6))
t = timed(lambda: h.copy_(d, non_blocking=True))
print("D2H alone   %.1f GB/s" % (n / t / 1e6))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timed(both)
print("H2D + D2H concurrent: %.1f GB/s each direction" % (n / t / 1e6))


# two H2D streams (two copy engines) against one D2H: does a second engine raise the
# aggregate when both directions run?
s3 = torch.cuda.Stream()
half = n // 2


def both2():
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        d[half:].copy_(h[half:], non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    for s in (s1, s2, s3):
        torch.cuda.current_stream().wait_stream(s)


t = timed(both2)
print("2x H2D (halves) + D2H concurrent: %.1f GB/s each direction" % (n / t / 1e6))


def h2d2():
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        d[half:].copy_(h[half:], non_blocking=True)
    for s in (s1, s3):
        torch.cuda.current_stream().wait_stream(s)


t = timed(h2d2)
print("2x H2D (halves) alone: %.1f GB/s" % (n / t / 1e6))
