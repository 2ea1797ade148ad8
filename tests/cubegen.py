# SPDX-License-Identifier: Apache-2.0
"""Seeded candidate generators for parity tests (numpy, host side).

Cubes use the xe_cube layout (include/xengine_b200.h): per candidate the R
cube then the S cube, each [D][T][W] uint32 words, W = ceil(T/32).
"""
from __future__ import annotations

import numpy as np


def words(T):
    return (T + 31) // 32


def pack(Rb: np.ndarray, Sb: np.ndarray) -> np.ndarray:
    """Rb, Sb: bool [n][D][T][T] -> uint32 [n][2*D*T*W]."""
    n, D, T, _ = Rb.shape
    W = words(T)
    pad = W * 32 - T
    bits = np.stack([Rb, Sb], axis=1)  # n,2,D,T,T
    if pad:
        bits = np.concatenate([bits, np.zeros(bits.shape[:-1] + (pad,), bool)], axis=-1)
    bits = bits.reshape(n, 2, D, T, W, 32).astype(np.uint64)
    w = (bits << np.arange(32, dtype=np.uint64)).sum(axis=-1).astype(np.uint32)
    return w.reshape(n, -1)


def unpack(cubes: np.ndarray, D: int, T: int):
    W = words(T)
    c = cubes.reshape(-1, 2, D, T, W).astype(np.uint64)
    bits = ((c[..., None] >> np.arange(32, dtype=np.uint64)) & 1).astype(bool)
    bits = bits.reshape(-1, 2, D, T, W * 32)[..., :T]
    return bits[:, 0], bits[:, 1]


def last_consumer(T, src, dst):
    last = np.full(T, -1)
    for s, d in zip(src, dst):
        last[s] = max(last[s], d)
    return last


def placement_cubes(a, dev: np.ndarray, policy=1):
    """dev [n][T] -> (Rb, Sb): save-all (policy 0) or minimal-save (1)."""
    n, T = dev.shape
    D = a.D
    last = last_consumer(T, a.src, a.dst) if policy == 1 else np.full(T, T - 1)
    Rb = np.zeros((n, D, T, T), bool)
    Sb = np.zeros((n, D, T, T), bool)
    ar = np.arange(n)
    for i in range(T):
        Rb[ar, dev[:, i], i, i] = True
        for t in range(i + 1, last[i] + 1):
            Sb[ar, dev[:, i], t, i] = True
    return Rb, Sb


def random_placements(a, n, rng, pin_input=True):
    dev = rng.integers(0, a.D, size=(n, a.T)).astype(np.uint8)
    if pin_input:
        # ops with a prohibitive cost somewhere go to their cheapest device
        for i in range(a.T):
            if (a.cost[:, i] >= 1e9).any():
                dev[:, i] = int(np.argmin(a.cost[:, i]))
    return dev


def recompute_edit(a, Rb, Sb, dev, rng, parents, consumers):
    """One drop-and-recompute edit per candidate row, valid for EQ11/EQ12."""
    n, D, T, _ = Rb.shape
    for c in range(n):
        cands = [i for i in range(T) if any(v > i + 1 for v in consumers[i])]
        if not cands:
            continue
        i = int(rng.choice(cands))
        t = int(rng.choice([v for v in consumers[i] if v > i + 1]))
        before = [v for v in consumers[i] if v < t]
        a0 = max([i + 1] + [v + 1 for v in before])
        if a0 > t:
            continue
        a1 = int(rng.integers(a0, t + 1))
        di = int(dev[c, i])
        dn = int(rng.integers(0, D)) if rng.random() < 0.5 else int(dev[c, t])
        if a.cost[dn, i] >= 1e9:
            dn = di
        Sb[c, di, a1:t + 1, i] = False
        Rb[c, dn, t, i] = True
        if Sb[c, di, t + 1:, i].any():
            rest = Sb[c, di, t + 1:, i].copy()
            Sb[c, di, t + 1:, i] = False
            Sb[c, dn, t + 1:, i] = rest
        for p in parents[i]:
            if Rb[c, :, t, p].any() or Sb[c, :, t, p].any():
                continue
            dp = int(dev[c, p])
            last_saved = p
            for tt in range(p + 1, t + 1):
                if Sb[c, dp, tt, p]:
                    last_saved = tt
            if Rb[c, dp, :, p].any() or last_saved >= p:
                Sb[c, dp, last_saved + 1:t + 1, p] = True


def adjacency(a):
    parents = [[] for _ in range(a.T)]
    consumers = [[] for _ in range(a.T)]
    for s, d in zip(a.src.tolist(), a.dst.tolist()):
        parents[d].append(s)
        consumers[s].append(d)
    return parents, consumers


def mixed_cubes(a, n, seed, edits=2, perturb=0.1, random_frac=0.05):
    """Placement + minimal-save + recompute edits (valid by construction),
    a fraction with single random bit flips, a fraction fully random."""
    rng = np.random.default_rng(seed)
    D, T = a.D, a.T
    dev = random_placements(a, n, rng)
    Rb, Sb = placement_cubes(a, dev, policy=1)
    parents, consumers = adjacency(a)
    for _ in range(edits):
        sel = rng.random(n) < 0.6
        idx = np.nonzero(sel)[0]
        if len(idx):
            r, s = Rb[idx], Sb[idx]
            recompute_edit(a, r, s, dev[idx], rng, parents, consumers)
            Rb[idx], Sb[idx] = r, s
    flip = rng.random(n) < perturb
    for c in np.nonzero(flip)[0]:
        which = rng.integers(0, 2)
        d, t, i = rng.integers(0, D), rng.integers(0, T), rng.integers(0, T)
        arr = Rb if which == 0 else Sb
        arr[c, d, t, i] = ~arr[c, d, t, i]
    rnd = rng.random(n) < random_frac
    k = int(rnd.sum())
    if k:
        dens = rng.random((k, 1, 1, 1)) * 0.3
        Rb[rnd] = rng.random((k, D, T, T)) < dens
        Sb[rnd] = rng.random((k, D, T, T)) < dens
    return pack(Rb, Sb)
