"""Executable model of the k_engine protocol (pm_engine.cu), for CPU tests.

Each in-flight region is a Python generator that yields at every point where
the device code spins (reader wait, landing wait, threshold wait, space wait)
and at the points where device threads of other CTAs may interleave.  A
scheduler runs W regions at a time and steps a random runnable one, so the
tests explore many interleavings of exactly the rules the kernel implements:

  * two-front ticket order (TwoFront in pm_engine.cuh),
  * gather: wait until the unit's location is a region of order >= t (or scratch),
  * publish reads; the last consumer frees the unit's slot / scratch unit,
  * occupants: wait for landing, wait for reads by consumers of order <= t,
    then (if still alive) take scratch first, else a free slot, copy, publish,
  * merge (stable, A wins ties) and write the region's slots.

The data really moves (numpy), so the final array is checked bit for bit.
"""

from __future__ import annotations

import random

import numpy as np

FREE, CLOSED = -1, -2


class TwoFront:
    def __init__(self, Q, qc):
        self.Q, self.qc = Q, qc

    def region_of_ticket(self, t):
        Q, qc = self.Q, self.qc
        if t == 0:
            return qc
        nl, nr = qc, Q - 1 - qc
        m2 = min(nl, nr)
        if t <= 2 * m2:
            return qc - (t + 1) // 2 if t & 1 else qc + t // 2
        return qc - (t - nr) if nl > nr else qc + (t - nl)

    def order(self, q):
        Q, qc = self.Q, self.qc
        if q == qc:
            return 0
        nl, nr = qc, Q - 1 - qc
        m2 = min(nl, nr)
        if q < qc:
            i = qc - q
            return 2 * i - 1 if i <= m2 else i + nr
        i = q - qc
        return 2 * i if i <= m2 else i + nl

    def window(self, t):
        nl, nr = self.qc, self.Q - 1 - self.qc
        m2 = min(nl, nr)
        if t <= 2 * m2:
            a, b = (t + 1) // 2, t // 2
        elif nl > nr:
            a, b = t - nr, nr
        else:
            a, b = nl, t - nl
        return self.qc - min(a, nl), self.qc + min(b, nr)


class NoSpace(Exception):
    pass


class EngineModel:
    def __init__(self, keys, payload, s, m, e, T, mu, scratch_units, mode="merge"):
        self.keys, self.pay = keys, payload
        self.s, self.m, self.e = s, m, e
        self.T, self.mu, self.M = T, mu, T * mu
        self.mode = mode
        self.k0 = s // T
        self.K = (e - 1) // T - self.k0 + 1
        self.R0 = s // self.M
        self.Q = (e - 1) // self.M - self.R0 + 1
        self.qc = min(max(m // self.M - self.R0, 0), self.Q - 1)
        self.tf = TwoFront(self.Q, self.qc)
        la, lb = m - s, e - m
        self.split = []
        A, B = keys[s:m], keys[m:e]
        for q in range(self.Q + 1):
            d = self.diag(q)
            if mode == "merge":  # stable merge path (A wins ties)
                lo, hi = max(0, d - lb), min(d, la)
                while lo < hi:
                    mid = (lo + hi) // 2
                    if A[mid] <= B[d - 1 - mid]:
                        lo = mid + 1
                    else:
                        hi = mid
                self.split.append(lo)
            else:
                self.split.append(min(max(d - lb, 0), la))
        self.state = list(range(self.K))
        self.loc = list(range(self.K))
        self.reads = [0] * self.K
        self.free_slots: list[int] = []
        self.free_scr = list(range(scratch_units))
        self.scr_k = np.zeros((scratch_units, T), keys.dtype)
        self.scr_p = np.zeros((scratch_units, T, payload.shape[1]), np.uint8)
        self.salvaged = 0

    # ---- geometry (Geo in pm_engine.cu) ----
    def slot_lo(self, j):
        return max(self.s, (self.k0 + j) * self.T)

    def slot_hi(self, j):
        return min(self.e, (self.k0 + j + 1) * self.T)

    def slot_base(self, j):
        return (self.k0 + j) * self.T

    def region_of_slot(self, j):
        return (self.k0 + j) // self.mu - self.R0

    def diag(self, q):
        if q <= 0:
            return 0
        if q >= self.Q:
            return self.e - self.s
        return (self.R0 + q) * self.M - self.s

    def consumed_by_window(self, j, t):
        wl, wr = self.tf.window(t)
        a_lo, a_hi = self.split[wl], self.split[wr + 1]
        b_lo, b_hi = self.diag(wl) - a_lo, self.diag(wr + 1) - a_hi
        x0, x1 = self.slot_lo(j), self.slot_hi(j)
        c = 0
        ua0, ua1 = x0 - self.s, min(x1, self.m) - self.s
        if ua1 > ua0:
            c += max(0, min(ua1, a_hi) - max(ua0, a_lo))
        ub0, ub1 = max(x0, self.m) - self.m, x1 - self.m
        if ub1 > ub0:
            c += max(0, min(ub1, b_hi) - max(ub0, b_lo))
        return c

    # ---- unit data access ----
    def read_unit(self, j, x0, x1):
        l, hb = self.loc[j], self.slot_base(j)
        if l >= 0:
            b = self.slot_base(l) + (x0 - hb)
            return self.keys[b:b + x1 - x0].copy(), self.pay[b:b + x1 - x0].copy()
        si = -l - 1
        return (self.scr_k[si, x0 - hb:x1 - hb].copy(), self.scr_p[si, x0 - hb:x1 - hb].copy())

    def free_location(self, j):
        l = self.loc[j]
        if l < 0:
            self.free_scr.append(-l - 1)
        elif self.slot_hi(l) - self.slot_lo(l) == self.T and self.state[l] == j:
            self.state[l] = FREE
            self.free_slots.append(l)

    # ---- one region, as a generator of wait points ----
    def region(self, t):
        q = self.tf.region_of_ticket(t)
        j0 = max(0, (self.R0 + q) * self.mu - self.k0)
        j1 = min(self.K, (self.R0 + q + 1) * self.mu - self.k0)
        occ = []
        for j in range(j0, j1):
            occ.append(self.state[j])
            self.state[j] = CLOSED
        d0, d1 = self.diag(q), self.diag(q + 1)
        a0, a1 = self.split[q], self.split[q + 1]
        b0, b1 = d0 - a0, d1 - a1
        la = self.m - self.s
        if self.mode == "merge" and ((a0 == d0 and a1 == d1) or (a0 == la and a1 == la)):
            return
        yield
        xa, xb = self.s + a0, self.m + b0
        pieces = []
        for run0, run1 in ((xa, self.s + a1), (xb, self.m + b1)):
            if run1 > run0:
                for j in range(run0 // self.T - self.k0, (run1 - 1) // self.T - self.k0 + 1):
                    pieces.append((j, max(run0, self.slot_lo(j)), min(run1, self.slot_hi(j)), run0 == xa))
        got = {}
        for j, x0, x1, isA in pieces:  # gather
            while True:
                l = self.loc[j]
                if l < 0 or self.tf.order(self.region_of_slot(l)) >= t:
                    break
                yield "wait"
            got[(j, isA)] = self.read_unit(j, x0, x1)
            yield
        for j, x0, x1, isA in pieces:  # publish reads
            self.reads[j] += x1 - x0
            if self.reads[j] == self.slot_hi(j) - self.slot_lo(j):
                self.free_location(j)
        yield
        for i, u in enumerate(occ):  # occupants
            if u < 0:
                continue
            slot = j0 + i
            while self.loc[u] != slot:
                yield "wait"
            thr = self.consumed_by_window(u, t)
            while self.reads[u] < thr:
                yield "wait"
            if self.reads[u] >= self.slot_hi(u) - self.slot_lo(u):
                continue
            spins = 0
            while True:
                if self.free_scr:
                    dest = -self.free_scr.pop() - 1
                    break
                f = None
                while self.free_slots:
                    f = self.free_slots.pop()
                    if self.state[f] == FREE:
                        self.state[f] = u
                        break
                    f = None
                if f is not None:
                    dest = f
                    break
                spins += 1
                if spins > 10000:
                    raise NoSpace(f"ticket {t} found no salvage space")
                yield "wait"
            x0, x1, hb = self.slot_lo(u), self.slot_hi(u), self.slot_base(u)
            sb = self.slot_base(slot) + (x0 - hb)
            k, p = self.keys[sb:sb + x1 - x0].copy(), self.pay[sb:sb + x1 - x0].copy()
            yield
            if dest >= 0:
                db = self.slot_base(dest) + (x0 - hb)
                self.keys[db:db + x1 - x0], self.pay[db:db + x1 - x0] = k, p
            else:
                self.scr_k[-dest - 1, x0 - hb:x1 - hb], self.scr_p[-dest - 1, x0 - hb:x1 - hb] = k, p
            self.loc[u] = dest
            self.salvaged += 1
        yield
        ka = np.concatenate([got[(j, True)][0] for j, _, _, isA in pieces if isA] or [self.keys[:0]])
        pa = np.concatenate([got[(j, True)][1] for j, _, _, isA in pieces if isA] or [self.pay[:0]])
        kb = np.concatenate([got[(j, False)][0] for j, _, _, isA in pieces if not isA] or [self.keys[:0]])
        pb = np.concatenate([got[(j, False)][1] for j, _, _, isA in pieces if not isA] or [self.pay[:0]])
        if self.mode == "merge":
            tag = np.concatenate([np.zeros(len(ka), np.int8), np.ones(len(kb), np.int8)])
            order = np.lexsort((tag, np.concatenate([ka, kb])))  # stable: key, then A before B
        else:
            order = np.concatenate([np.arange(len(ka), len(ka) + len(kb)), np.arange(len(ka))])
        kk = np.concatenate([ka, kb])[order]
        pp = np.concatenate([pa, pb])[order]
        o0 = self.s + d0
        self.keys[o0:o0 + len(kk)] = kk
        self.pay[o0:o0 + len(kk)] = pp

    def run(self, inflight, rng: random.Random):
        """Run all tickets with `inflight` concurrent regions under a random scheduler."""
        nxt, active = 0, []
        waits = 0
        while nxt < self.Q or active:
            while len(active) < inflight and nxt < self.Q:
                active.append(self.region(nxt))
                nxt += 1
            gen = rng.choice(active)
            try:
                r = next(gen)
                if r == "wait":
                    waits += 1
                    if waits > 10_000_000:
                        raise RuntimeError("model livelock")
            except StopIteration:
                active.remove(gen)
        return self
