import numpy as np, sys
rng = np.random.default_rng(0)
def make(N, kind="uniform"):
    L = N//2
    if kind == "uniform":
        a = np.sort(rng.integers(0, 2**31, L)); b = np.sort(rng.integers(0, 2**31, L))
    elif kind == "dup":
        a = np.sort(rng.integers(0, 1024, L)); b = np.sort(rng.integers(0, 1024, L))
    return a, b
def splits(a, b, T):
    N = len(a)+len(b); K = N//T
    # merge path: for diag d, a_d = number of A among first d outputs (A wins ties)
    keys = np.concatenate([a, b]); src = np.concatenate([np.zeros(len(a),np.int8), np.ones(len(b),np.int8)])
    order = np.argsort(keys, kind="stable")
    isA = (src[order] == 0)
    ca = np.concatenate([[0], np.cumsum(isA)])
    d = np.arange(K+1)*T
    return ca[d], d - ca[d], order
def graph(a, b, T):
    LA = len(a); N = LA+len(b); K = N//T
    sa, sb, order = splits(a, b, T)
    # dest[y] = output position of record at position y
    dest = np.empty(N, np.int64); dest[order] = np.arange(N)
    reader = dest // T   # region reading record at y
    block = np.arange(N)//T
    # edges (block p, region r, count)
    key = block*K + reader
    u, cnt = np.unique(key, return_counts=True)
    return u//K, u%K, cnt, reader, K
def evaluate(name, t, p, r, c, K, T, W=1000):
    # t: rank of region in processing order (0..K-1)
    m = p != r
    sal = m & (t[r] > t[p])
    sv = c[sal].sum()/ (K*T)
    # live pool: salvage of (p->r) lives [t[p], t[r]]
    ev = np.zeros(K+1)
    np.add.at(ev, t[p[sal]], c[sal]); np.add.at(ev, t[r[sal]], -c[sal])
    live = np.cumsum(ev)[:-1].max()/(K*T)
    # slack of non-salvage edges
    ok = m & (t[r] < t[p])
    gap = t[p[ok]] - t[r[ok]]
    tight = (gap < W).mean()
    print(f"{name:28s} salvage={sv:.3f}N  peak_live={live:.3f}N  tight_edges(<{W})={tight:.3f}  block_salv_frac={len(np.unique(p[sal]))/K:.3f}")
def itin_angle(reader, K, T, n, LAblocks):
    # itinerary of block p: side(p), side(D(p)), ... where D(p)=reader of p's middle record
    mid = np.arange(K)*T + T//2
    Dblk = reader[mid]   # region index reading middle of block p
    w = np.exp(2j*np.pi*np.arange(1, n+1)/n)
    z = np.zeros(K, complex); cur = np.arange(K)
    for i in range(n):
        bit = (cur >= LAblocks).astype(float)
        z += bit*w[i]
        cur = Dblk[cur]
    return np.angle(z), np.abs(z)
def rank(v):
    t = np.empty(len(v), np.int64); t[np.argsort(v, kind="stable")] = np.arange(len(v)); return t
if __name__ == "__main__":
    N = 1 << int(sys.argv[1]); T = 1 << int(sys.argv[2]); kind = sys.argv[3] if len(sys.argv) > 3 else "uniform"
    a, b = make(N, kind)
    p, r, c, reader, K = graph(a, b, T)
    n = int(np.log2(K))
    print("K", K, "n", n, "edges", len(p))
    q = np.arange(K)
    # two-front: distance from boundary
    mid = K//2
    evaluate("ascending", q, p, r, c, K, T)
    evaluate("two-front", rank(np.abs(q + 0.5 - mid)), p, r, c, K, T)
    for nn in [n, n+2, n+4, n-2]:
        ang, mag = itin_angle(reader, K, T, nn, K//2)
        for off in [0.0, np.pi/2, np.pi, -np.pi/2]:
            v = np.mod(ang - off, 2*np.pi)
            evaluate(f"angle n={nn} off={off:.2f}", rank(v), p, r, c, K, T)
