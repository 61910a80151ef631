import sys, faulthandler, torch
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
_ops.set_engine_only(True)
for L in [int(x) for x in sys.argv[2:]]:
    k0, p0, m = config_input_device(2, seed=3, log_len=L)
    n = k0.numel()
    ref = torch.sort(k0, stable=True).values
    _ops.set_flow_mode(sys.argv[1])
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    print("L", L, "start", flush=True)
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n)
        print("launched", flush=True)
        torch.cuda.synchronize()
        print("synced", flush=True)
    print("L", L, sys.argv[1], torch.equal(arr.keys, ref), flush=True)
