"""Readers for the committed reference fixtures (tests/golden/*.npz)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def merge_cases(name="merge_i32.npz"):
    z = load(name)
    for i in range(int(z["count"])):
        p = f"c{i}_"
        yield {k[len(p):]: z[k] for k in z.files if k.startswith(p)}


def median_cases():
    z = load("median.npz")
    a, b, pa, pb, piv = z["a"], z["b"], z["pos_a"], z["pos_b"], z["pivots"]
    for j in range(len(piv)):
        yield a[pa[j]:pa[j + 1]], b[pb[j]:pb[j + 1]], tuple(int(x) for x in piv[j])


def shift_cases():
    yield from merge_cases("shift.npz")


def plan_cases():
    z = load("plan.npz")
    for i in range(int(z["count"])):
        p = f"c{i}_"
        d = {k[len(p):]: z[k] for k in z.files if k.startswith(p)}
        inst = int(d["inst"])
        d["keys"] = z[f"i{inst}_keys"]
        d["payload"] = z[f"i{inst}_payload"]
        yield d


def big():
    z = load("big.npz")
    return {k: str(z[k]) for k in z.files}
