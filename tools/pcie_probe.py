"""PCIe probe: pinned 1 GiB host<->device copies, each direction alone and both
at once (the e2e ceiling of a sort that moves every key in and out)."""
import time

import torch

n = 1 << 28
h_in = torch.empty(n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n, dtype=torch.int32).pin_memory()
d_a = torch.empty(n, dtype=torch.int32, device="cuda")
d_b = torch.empty(n, dtype=torch.int32, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def run(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


gb = 4 * n / 1e9
t = run(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D alone {gb / t:.1f} GB/s")
t = run(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H alone {gb / t:.1f} GB/s")


def both():
    with torch.cuda.stream(up):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(down):
        h_out.copy_(d_b, non_blocking=True)


t = run(both)
print(f"both at once: {gb / t:.1f} GB/s each direction ({t * 1e3:.1f} ms per 1 GiB each way)")
for chunks in (4, 16):
    def chunked():
        m = n // chunks
        for c in range(chunks):
            with torch.cuda.stream(up):
                d_a[c * m:(c + 1) * m].copy_(h_in[c * m:(c + 1) * m], non_blocking=True)
            with torch.cuda.stream(down):
                h_out[c * m:(c + 1) * m].copy_(d_b[c * m:(c + 1) * m], non_blocking=True)
    t = run(chunked)
    print(f"both, {chunks} interleaved chunks: {gb / t:.1f} GB/s each direction")

# two copy streams per direction (halves): does a second copy engine help?
up2, down2 = torch.cuda.Stream(), torch.cuda.Stream()


def both_two_engines():
    m = n // 2
    for s_up, s_dn, c in ((up, down, 0), (up2, down2, 1)):
        with torch.cuda.stream(s_up):
            d_a[c * m:(c + 1) * m].copy_(h_in[c * m:(c + 1) * m], non_blocking=True)
        with torch.cuda.stream(s_dn):
            h_out[c * m:(c + 1) * m].copy_(d_b[c * m:(c + 1) * m], non_blocking=True)


t = run(both_two_engines)
print(f"both, two streams per direction: {gb / t:.1f} GB/s each direction")


def h2d_two_engines():
    m = n // 2
    for s_up, c in ((up, 0), (up2, 1)):
        with torch.cuda.stream(s_up):
            d_a[c * m:(c + 1) * m].copy_(h_in[c * m:(c + 1) * m], non_blocking=True)


t = run(h2d_two_engines)
print(f"H2D alone, two streams: {gb / t:.1f} GB/s")
