"""Quick GPU bring-up script: small merges with progressively larger sizes."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from oracle import oracle as orc
rng = np.random.default_rng(0)
for size, dom, w in [(10, 5, 0), (100, 50, 4), (9000, 100, 0), (20000, 10**6, 4), (100000, 1000, 0), (1 << 20, 2**31-1, 0), (1 << 21, 1024, 4)]:
    m = size // 2
    a = np.sort(rng.integers(0, dom, m)).astype(np.int32); b = np.sort(rng.integers(0, dom, size - m)).astype(np.int32)
    k = np.concatenate([a, b]); p = rng.integers(0, 256, (size, w), dtype=np.uint8)
    wk, wp = k.copy(), p.copy(); orc.seq_merge_buffered(wk, wp, 0, m, size)
    arr = pm.KeyedArray(torch.from_numpy(k).cuda(), torch.from_numpy(p).cuda())
    t0 = time.time()
    try:
        pm.merge_srecpar(arr, pm.MergeJob(0, m, size), 8)
    except Exception as ex:
        print('FAIL', size, dom, w, ex); sys.stdout.flush(); continue
    gk, gp = arr.numpy()
    ok = np.array_equal(gk, wk) and np.array_equal(gp, wp)
    bad = np.flatnonzero(gk != wk)
    print(size, dom, w, 'ok' if ok else f'MISMATCH first={bad[:5]} n={len(bad)}', f'{time.time()-t0:.3f}s', pm.synchronize()); sys.stdout.flush()
