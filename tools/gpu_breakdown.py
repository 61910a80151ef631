import sys, time
import torch
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); sizes = [int(x) for x in sys.argv[2].split(',')]
scr_div = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 7
names = ['d_gather', 'd_land', 'd_publish', 'd_merge', 'd_waitdefer', 'd_store']
for L in sizes:
    kw = {"log_len_b": 16} if cfg == 3 else {}
    k0, p0, m = config_input_device(cfg, seed=1, log_len=L, **kw)
    times = []
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(reps):
        arr.keys.copy_(k0)
        if p0.shape[1]:
            arr.payload.copy_(p0)
        torch.cuda.synchronize()
        e0.record()
        with pm.deferred_checks():
            _ops.merge(arr, 0, m, len(k0), scratch_records=(len(k0) // scr_div if scr_div else 0))
        e1.record()
        st = pm.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    times.sort()
    dt = times[len(times) // 2]
    nr = max(st[2] + st[3], 1)
    br = ' '.join(f"{n}={st[4+i]/nr:.0f}" for i, n in enumerate(names)) + f" s_step1={st[10]/nr:.0f} s_step2={st[11]/nr:.0f}"
    tot = 1
    print(f"L={L} med {dt*1e3:.3f}ms min {times[0]*1e3:.3f}ms salv_units={st[0]} salv_frac={st[1]/len(k0):.3f} regions={st[2]} ident={st[3]} "
          f"(cycles per region, CTA-summed) {br} "
          f"salvage-split(warp-cycles): land={st[12]:.3g} thr={st[13]:.3g} dest={st[14]:.3g} copy={st[15]:.3g}", flush=True)
