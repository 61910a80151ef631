"""PCIe rates of chunked copies (the pm_merge_host pattern): 96 chunks of the
4 GiB record array, H2D alone, D2H alone, both directions at once on two
streams, and both with 8 host threads copying pinned memory at the same time."""
import threading
import time

import numpy as np
import torch

n = 4 << 30
nch = 96
c = n // nch
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, down, same_buffer=False, host_threads=0):
    torch.cuda.synchronize()
    stop = threading.Event()
    th = []
    if host_threads:
        a = torch.empty(256 << 20, dtype=torch.uint8).pin_memory().numpy()
        b = torch.empty(256 << 20, dtype=torch.uint8).pin_memory().numpy()

        def spin():
            while not stop.is_set():
                np.copyto(b, a)
        th = [threading.Thread(target=spin) for _ in range(host_threads)]
        [t.start() for t in th]
    t0 = time.perf_counter()
    dst = h_src if same_buffer else h_dst
    for k in range(nch):
        if up:
            with torch.cuda.stream(s1):
                d_a[k * c:(k + 1) * c].copy_(h_src[k * c:(k + 1) * c], non_blocking=True)
        if down:
            with torch.cuda.stream(s2):
                dst[k * c:(k + 1) * c].copy_(d_b[k * c:(k + 1) * c], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    stop.set()
    [t.join() for t in th]
    return n / dt / 1e9


for name, kw in (("H2D", dict(up=1, down=0)), ("D2H", dict(up=0, down=1)), ("both", dict(up=1, down=1)),
                 ("both, same host buffer", dict(up=1, down=1, same_buffer=True)),
                 ("both + 4 host memcpy threads", dict(up=1, down=1, host_threads=4)),
                 ("both + 8 host memcpy threads", dict(up=1, down=1, host_threads=8))):
    r = [run(**kw) for _ in range(3)]
    print(f"{name:30s} {max(r):6.1f} GB/s per direction", flush=True)
