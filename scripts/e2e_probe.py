"""Where the end-to-end (host buffer) time goes for a workload: pinned H2D
alone, device decode alone, decode_host (chunked, two streams)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1202_1060_b200 as P  # noqa: E402
import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_n64800"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
g, s, ebn0, _ = bench.workload(name)
n = g.n_vars
llr = P.transmit_all_zero(n, P.sigma2_from_ebn0(ebn0, g.rate), 1, 0, B)
h = torch.empty((B, n), dtype=torch.float32, pin_memory=True)
h.copy_(llr.cpu())
d = torch.empty_like(llr)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print(f"{name} B={B} plan={P.plan(g, s, B)}")
print(f"H2D pinned {B * n * 4 / 1e9:.2f} GB: {timed(lambda: d.copy_(h, non_blocking=True)):.1f} ms")
print(f"decode_device: {timed(lambda: P.decode_batch(g, s, llr, 10, early_stop=False, packed=True)):.1f} ms")
bits = torch.empty((B, (n + 7) // 8), dtype=torch.uint8, pin_memory=True)
cnt = torch.zeros(6, dtype=torch.int64)
print(f"decode_host: {timed(lambda: P.decode_host(g, s, h, 10, early_stop=False, packed=True, bits=bits, counters=cnt)):.1f} ms")

# chunk-size effects on the device path
half = B // 2
a = llr[:half].contiguous()
b = llr[half:].contiguous()
print(f"decode_device {half}: {timed(lambda: P.decode_batch(g, s, a, 10, early_stop=False, packed=True)):.1f} ms")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    with torch.cuda.stream(s1):
        P.decode_batch(g, s, a, 10, early_stop=False, packed=True)
    with torch.cuda.stream(s2):
        P.decode_batch(g, s, b, 10, early_stop=False, packed=True)


print(f"2 x decode_device {half} on two streams: {timed(two):.1f} ms")


def seq_h2d():
    da = torch.empty_like(a)
    db = torch.empty_like(b)
    with torch.cuda.stream(s1):
        da.copy_(h[:half], non_blocking=True)
        P.decode_batch(g, s, da, 10, early_stop=False, packed=True)
    with torch.cuda.stream(s2):
        db.copy_(h[half:], non_blocking=True)
        P.decode_batch(g, s, db, 10, early_stop=False, packed=True)


print(f"H2D+decode halves on two streams: {timed(seq_h2d):.1f} ms")
