"""Executable model of the k_engine protocol (pm_engine.cu), for CPU tests.

Each in-flight ticket is a set of Python generators -- one salvage item per
slot of its region and one data phase -- that yield at every point where the
device code spins (reader wait, landing wait, space wait, item wait, consumer
wait) and where threads of other CTAs may interleave.  A scheduler keeps W
tickets in flight and steps a random runnable generator, so the tests explore
many interleavings of exactly the rules the kernel implements:

  * two-front ticket order (TwoFront in pm_engine.cuh),
  * salvage item: close the slot, wait for its occupant to land, and if a region
    of higher order still needs it, move it (scratch first, else a free slot;
    no space -> wait for the ticket's reads to be published, then block),
  * data: gather (wait until each unit sits in a region of order >= t or in
    scratch), publish reads (the last consumer frees the unit's location), merge
    (stable, A wins ties), wait for every slot item and for every consumer of
    order <= t to have read each occupant, then write the region's slots.

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
    def read_unit(self, j, x0, x1, l=None):
        l = self.loc[j] if l is None else l
        hb = self.slot_base(j)
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

    # ---- one ticket: slot items + the data phase, as generators of wait points ----
    def ticket(self, t):
        """Return the generators of ticket t (k_engine in pm_engine.cu): one salvage
        item per slot of its region, and the data phase."""
        q = self.tf.region_of_ticket(t)
        j0 = max(0, (self.R0 + q) * self.mu - self.k0)
        j1 = min(self.K, (self.R0 + q + 1) * self.mu - self.k0)
        d0, d1 = self.diag(q), self.diag(q + 1)
        a0, a1 = self.split[q], self.split[q + 1]
        la = self.m - self.s
        identity = self.mode == "merge" and ((a0 == d0 and a1 == d1) or (a0 == la and a1 == la))
        st = {"items_done": 0, "published": False, "occ": [-1] * (j1 - j0)}

        def item(i):
            slot = j0 + i
            u = self.state[slot]  # close the slot (atomicExch) and sample its occupant
            self.state[slot] = CLOSED
            yield
            if u >= 0 and not identity:
                st["occ"][i] = u
                while self.loc[u] != slot:  # landing: the mover has published
                    yield "wait"
                if self.consumed_by_window(u, t) < self.slot_hi(u) - self.slot_lo(u):
                    # a later region still needs u: move it now (no wait for earlier
                    # consumers -- they read either copy; the data phase waits for them)
                    dest = self.take_space(u, t, block=False)
                    if dest is None:
                        while not st["published"]:  # the region's own reads free space first
                            yield "wait"
                        spins = 0
                        while (dest := self.take_space(u, t, block=True)) is None:
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
                    yield
                    self.loc[u] = dest  # publish (after the copy is visible)
                    self.salvaged += 1
            st["items_done"] += 1

        def data():
            if identity:
                st["published"] = True
                while st["items_done"] < j1 - j0:
                    yield "wait"
                return
            yield
            xa, xb = self.s + a0, self.m + (d0 - a0)
            b1 = d1 - a1
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
                yield  # the bulk copy reads the location seen above, later (TMA is asynchronous)
                got[(j, isA)] = self.read_unit(j, x0, x1, l)
                yield
            last = []
            for j, x0, x1, isA in pieces:  # publish reads
                self.reads[j] += x1 - x0
                if self.reads[j] == self.slot_hi(j) - self.slot_lo(j):
                    last.append(j)
            st["published"] = True
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
            yield
            for j in last:  # last reader frees the unit's location
                self.free_location(j)
            yield
            while st["items_done"] < j1 - j0:  # every slot item is done
                yield "wait"
            for u in st["occ"]:  # every consumer of order <= t has read each occupant
                if u >= 0:
                    while self.reads[u] < self.consumed_by_window(u, t):
                        yield "wait"
            o0 = self.s + d0
            self.keys[o0:o0 + len(kk)] = kk
            self.pay[o0:o0 + len(kk)] = pp

        return [item(i) for i in range(j1 - j0)] + [data()]

    def take_space(self, u, t, block):
        """Scratch first, then a free slot of a region of order > t (acquire_dest:
        units only move to higher order, so reads[u] counts exactly the consumers
        of order <= r while u sits in region r); None if there is none."""
        if self.free_scr:
            return -self.free_scr.pop() - 1
        while self.free_slots:
            f = self.free_slots.pop()
            if self.state[f] == FREE and self.tf.order(self.region_of_slot(f)) > t:
                self.state[f] = u
                return f
        return None

    def run(self, inflight, rng: random.Random):
        """Run all tickets with at most `inflight` unfinished tickets under a random scheduler."""
        nxt, active, tickets = 0, [], []
        waits = 0
        while nxt < self.Q or active:
            while len(tickets) < inflight and nxt < self.Q:
                gens = self.ticket(nxt)
                tickets.append(gens[-1])  # a ticket is finished when its data phase is
                active.extend(gens)
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
                if gen in tickets:
                    tickets.remove(gen)
        return self
