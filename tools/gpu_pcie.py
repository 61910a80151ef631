"""PCIe rates with pinned host buffers: H2D alone, D2H alone, both at once (two
streams), the e2e bound of pm_merge_host's in-place host semantics (1.25 N / R)."""
import torch

n = 1 << 30  # bytes per direction
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def h2d():
    d_a.copy_(h_src, non_blocking=True)


def d2h():
    h_dst.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D {n / t1 / 1e6:.1f} GB/s  D2H {n / t2 / 1e6:.1f} GB/s  both at once {n / t3 / 1e6:.1f} GB/s per direction")
for bytes_total in (4 << 30,):
    r = n / t3 / 1e6
    print(f"pm_merge_host bound for {bytes_total >> 30} GiB of records: 1.25 N / R = {1.25 * bytes_total / r / 1e6:.1f} ms "
          f"(R = {r:.1f} GB/s bidirectional)")
