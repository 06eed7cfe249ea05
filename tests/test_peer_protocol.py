"""CPU model check of the PEER backend's flag protocol (rvk_dcg.cu header).

Each rank runs the same kernel sequence per solve -- reset (seq += 1),
setup, [K1(it), K2(it)] x max_it, finish -- and every kernel is modelled as
  start : its flag wait (peer_wait tag) is satisfied; its reads open and must
          see the expected version of every region they read (RAW);
  write : its stores land in local and REMOTE regions (halo planes, gather
          slots); no other rank may hold an open read of a region it
          overwrites with a new version (WAR);
  end   : reads close, flag released on every rank (peer_publish).
A random scheduler interleaves the ranks; the test asserts no RAW/WAR
violation and no deadlock across repeated solves, and -- as a negative
control -- that dropping the setup's finish-barrier wait is caught.

Regions (per receiving rank q):  zh[q,side]  z halo plane from a neighbour,
ph[q,k,side]  halo plane of p buffer k, slot[q,src,'zz'|'pw']  gather slot.
Versions are (solve, iteration) pairs.
"""
import random

import pytest

FINISH = 0xFFFFFFFF


def tag(seq, phase):
    return (seq << 32) | phase


class Model:
    def __init__(self, P, max_it, solves, setup_barrier=True):
        self.P, self.max_it, self.solves = P, max_it, solves
        self.setup_barrier = setup_barrier
        self.flags = [[0] * P for _ in range(P)]     # flags[receiver][source]
        self.ver = {}                                # region -> version
        self.open_reads = {}                         # rank -> {region: version}
        self.prog = [self.program(r) for r in range(P)]
        self.pc = [0] * P
        self.state = ["idle"] * P                    # idle -> running -> idle

    # ---- what each kernel waits for / reads / writes (rvk_dcg.cu) ----------
    def nbrs(self, r):
        # (neighbour, side of the NEIGHBOUR's halo my boundary plane lands in)
        out = []
        if r > 0:
            out.append((r - 1, "hi"))
        if r < self.P - 1:
            out.append((r + 1, "lo"))
        return out

    def my_halos(self, r):
        return [s for s, ok in (("lo", r > 0), ("hi", r < self.P - 1)) if ok]

    def program(self, r):
        ops = []
        for s in range(1, self.solves + 1):
            # k_dcg_setup: waits every rank's finish(s-1) when s > 1
            wait = tag(s - 1, FINISH) if (s > 1 and self.setup_barrier) else 0
            writes = {("zh", q, side): (s, 0) for q, side in self.nbrs(r)}
            writes.update({("slot", q, r, "zz"): (s, 0) for q in range(self.P)})
            ops.append(("setup", wait, {}, writes, tag(s, 1)))
            for it in range(self.max_it):
                # K1(it): waits 2it+1; reads z halos (z_it), p_old halos (p_{it-1}),
                # zz slots (it); writes p_new halos into neighbours, pw slots
                reads = {("zh", r, side): (s, it) for side in self.my_halos(r)}
                if it > 0:
                    reads.update({("ph", r, it & 1, side): (s, it - 1) for side in self.my_halos(r)})
                reads.update({("slot", r, q, "zz"): (s, it) for q in range(self.P)})
                writes = {("ph", q, (it + 1) & 1, side): (s, it) for q, side in self.nbrs(r)}
                writes.update({("slot", q, r, "pw"): (s, it) for q in range(self.P)})
                ops.append((f"K1({it})", tag(s, 2 * it + 1), reads, writes, tag(s, 2 * it + 2)))
                # K2(it): waits 2it+2; reads pw slots; writes z_{it+1} halos, zz slots
                reads = {("slot", r, q, "pw"): (s, it) for q in range(self.P)}
                writes = {("zh", q, side): (s, it + 1) for q, side in self.nbrs(r)}
                writes.update({("slot", q, r, "zz"): (s, it + 1) for q in range(self.P)})
                ops.append((f"K2({it})", tag(s, 2 * it + 2), reads, writes, tag(s, 2 * it + 3)))
            reads = {("slot", r, q, "zz"): (s, self.max_it) for q in range(self.P)}
            ops.append(("finish", tag(s, 2 * self.max_it + 1), reads, {}, tag(s, FINISH)))
        return ops

    # ---- scheduler steps ----------------------------------------------------
    def enabled(self, r):
        if self.pc[r] >= len(self.prog[r]):
            return None
        name, wait, reads, writes, sig = self.prog[r][self.pc[r]]
        if self.state[r] == "idle":
            return "start" if all(f >= wait for f in self.flags[r]) else None
        return self.state[r]

    def step(self, r, errors):
        name, wait, reads, writes, sig = self.prog[r][self.pc[r]]
        if self.state[r] == "idle":
            for reg, v in reads.items():
                if self.ver.get(reg) != v:
                    errors.append(f"RAW: rank {r} {name} reads {reg} at {self.ver.get(reg)}, wants {v}")
            self.open_reads[r] = dict(reads)
            self.state[r] = "write"
        elif self.state[r] == "write":
            for reg, v in writes.items():
                for q, rd in self.open_reads.items():
                    if q != r and reg in rd and rd[reg] != v:
                        errors.append(f"WAR: rank {r} {name} overwrites {reg} (-> {v}) "
                                      f"while rank {q} reads version {rd[reg]}")
                self.ver[reg] = v
            self.state[r] = "end"
        else:  # end: reads close, flag released on every rank
            self.open_reads.pop(r, None)
            for q in range(self.P):
                assert sig >= self.flags[q][r], "flags must be monotone per source"
                self.flags[q][r] = sig
            self.state[r] = "idle"
            self.pc[r] += 1

    def run(self, rng):
        errors = []
        while True:
            ready = [r for r in range(self.P) if self.enabled(r)]
            if not ready:
                done = all(self.pc[r] >= len(self.prog[r]) for r in range(self.P))
                return errors, done
            self.step(rng.choice(ready), errors)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_peer_protocol_safe_and_live(P):
    for seed in range(60):
        m = Model(P, max_it=4, solves=3)
        errors, done = m.run(random.Random(seed * 7919 + P))
        assert done, f"deadlock (seed {seed})"
        assert not errors, errors[:3]


def test_peer_protocol_without_setup_barrier_is_caught():
    """Negative control: without setup(s) waiting for every finish(s-1), a
    fast rank overwrites a slow rank's zz slot before its finish read it."""
    caught = False
    for seed in range(400):
        m = Model(3, max_it=2, solves=3, setup_barrier=False)
        errors, done = m.run(random.Random(seed))
        if errors:
            caught = True
            break
    assert caught
