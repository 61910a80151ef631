"""A few in-place merges at 2^L records per side (default 22, 24) for ncu launch lists
of the medium-size paths."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2005_12648_b200 as pm  # noqa: E402
from paper_2005_12648_b200 import _ops  # noqa: E402
from paper_2005_12648_b200.workloads import config_input_device  # noqa: E402

for L in [int(x) for x in sys.argv[1:]] or [22, 24]:
    k0, p0, m = config_input_device(2, seed=3, log_len=L)
    arr = pm.KeyedArray(k0.clone(), p0.clone())
    for i in range(3):
        arr.keys.copy_(k0)
        with pm.deferred_checks():
            _ops.merge(arr, 0, m, k0.numel())
    torch.cuda.synchronize()
