import sys, statistics, torch
sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for L in (21, 22, 23, 24):
    k0, p0, m = config_input_device(2, seed=3, log_len=L)
    n = k0.numel()
    ref = torch.sort(k0).values
    res = {}
    for mode in ("staged", "buffered", "flow"):
        arr = pm.KeyedArray(k0.clone(), p0.clone())
        ts = []
        for i in range(8):
            arr.keys.copy_(k0)
            if mode != "staged":
                _ops.set_engine_only(True)
                _ops.set_flow_mode("bounded" if mode == "buffered" else "auto")
            torch.cuda.synchronize()
            e0.record()
            with pm.deferred_checks():
                _ops.merge(arr, 0, m, n, scratch_records=(min(m, n - m) if mode == "buffered" else 0))
            e1.record(); e1.synchronize()
            _ops.set_engine_only(False); _ops.set_flow_mode("auto")
            if i: ts.append(e0.elapsed_time(e1))
        ok = torch.equal(arr.keys, ref)
        res[mode] = (round(statistics.median(ts) * 1e3, 1), ok)
    print(L, res, flush=True)
