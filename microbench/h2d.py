"""Host->device copy bandwidth of a pinned 4 GiB buffer (the e2e ceiling)."""
import torch

n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.synchronize()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return n / (best * 1e-3) / 1e9


print("one copy      GB/s", round(timed(lambda: d.copy_(h, non_blocking=True)), 1))
for chunk in (64 << 20, 256 << 20, 512 << 20):
    def chunked(chunk=chunk):
        for o in range(0, n, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    print(f"chunks {chunk >> 20:4d} MiB GB/s", round(timed(chunked), 1))


def two_streams():
    half = n // 2
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)


print("two streams   GB/s", round(timed(two_streams), 1))
print("D2H one copy  GB/s", round(timed(lambda: h.copy_(d, non_blocking=True)), 1))
