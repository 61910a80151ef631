import sys, time
import torch
sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from paper_2005_12648_b200.workloads import config_input_device
cfg = int(sys.argv[1]); sizes = [int(x) for x in sys.argv[2].split(',')]
names = ['ticket', 'g_issue', 'g_land', 'salvage', 'merge', 'store']
for L in sizes:
    kw = {"log_len_b": 16} if cfg == 3 else {}
    k0, p0, m = config_input_device(cfg, seed=1, log_len=L, **kw)
    for rep in range(2):
        arr = pm.KeyedArray(k0.clone(), p0.clone())
        torch.cuda.synchronize(); t0 = time.time()
        with pm.deferred_checks():
            _ops.merge(arr, 0, m, len(k0))
        dt = time.time() - t0
        st = pm.synchronize()
    tot = sum(st[4:10])
    br = ' '.join(f"{n}={st[4+i]/tot*100:.1f}%" for i, n in enumerate(names))
    print(f"L={L} {dt*1e3:.2f}ms salv_units={st[0]} salv_frac={st[1]/len(k0):.3f} regions={st[2]} ident={st[3]} "
          f"cycles/region={tot/max(st[2]+st[3],1):.0f} {br} spins_r={st[10]} spins_o={st[11]} "
          f"salvage-split(warp-cycles): land={st[12]:.3g} thr={st[13]:.3g} dest={st[14]:.3g} copy={st[15]:.3g}", flush=True)
