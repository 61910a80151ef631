import sys
import torch, numpy as np
sys.path.insert(0, '.')  # run from the repo root
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops, _capi
from paper_2005_12648_b200.workloads import config_input_device
L = int(sys.argv[1])
k0, p0, m = config_input_device(2, seed=1, log_len=L)
n = len(k0); M = 8192
Q = (n - 1) // M + 1
diags = torch.tensor([min(q * M, n) for q in range(Q + 1)], dtype=torch.int64)
true = pm.find_splits(k0[:m], k0[m:], diags).cpu().numpy()
arr = pm.KeyedArray(k0.clone(), p0.clone())
try:
    with pm.deferred_checks():
        _ops.merge(arr, 0, m, n)
except Exception as ex:
    print("merge error", ex)
got = np.zeros(Q + 1, np.int64)
print(_capi.lib().pm_debug_splits(_capi.context(0), got.ctypes.data, Q + 1))
bad = np.flatnonzero(got != true)
print("Q", Q, "qc", min(m // M, Q - 1), "bad", len(bad), bad[:20], got[bad[:10]], true[bad[:10]])
qc = min(m // M, Q - 1)
for q in list(range(0, 6)) + list(range(qc - 460, qc - 440)) + list(range(qc + 440, qc + 460)) + list(range(Q - 4, Q + 1)):
    if 0 <= q <= Q:
        print(q, got[q], true[q], q * M)
badL = [q for q in range(qc, 0, -1) if got[q] != true[q]]
badR = [q for q in range(qc, Q) if got[q] != true[q]]
print("first bad going left", badL[:3], "going right", badR[:3], "look ~", 2 * 148 * 3)
if badL:
    q = badL[0]
    for x in range(q - 2, q + 4):
        print(x, got[x], true[x], x * M)
