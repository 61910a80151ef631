"""Bring-up: time each size with status checks; prints as it goes."""
import sys, time, ctypes
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _capi
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sizes = [int(x) for x in sys.argv[2].split(',')] if len(sys.argv) > 2 else [18, 20, 22, 24, 26, 28, 29]
for L in sizes:
    t0 = time.time()
    kw = {"log_len_b": 16} if cfg == 3 else {}
    k0, p0, m = config_input_device(cfg, seed=1, log_len=L, **kw)
    torch.cuda.synchronize()
    t1 = time.time()
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    torch.cuda.synchronize()
    t2 = time.time()
    try:
        with pm.deferred_checks():
            from paper_2005_12648_b200 import _ops
            _ops.merge(arr, 0, m, len(k0))
    except Exception as ex:
        print(f"L={L} FAILED after {time.time()-t2:.2f}s: {ex}", flush=True)
        break
    t3 = time.time()
    st = pm.synchronize()
    ok = bool(torch.all(arr.keys[1:] >= arr.keys[:-1]).item())
    print(f"L={L} gen {t1-t0:.2f}s merge {t3-t2:.3f}s ok={ok} stats={st} N={len(k0)}", flush=True)
