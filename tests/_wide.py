"""Wide-domain (NEXT-4, d > 64) test inputs: value duplication of one-word
instances and helpers to move between one-word and multi-word domain states.
Test-only constructors (no method arithmetic)."""
from __future__ import annotations

import numpy as np

import synth

U64 = np.uint64


def bits_of(D, n, wq):
    """[n, 64*wq] bool view of a wide domain state."""
    D = np.asarray(D, dtype=U64).reshape(n, wq)
    out = np.zeros((n, 64 * wq), dtype=bool)
    for w in range(wq):
        for b in range(64):
            out[:, 64 * w + b] = ((D[:, w] >> U64(b)) & U64(1)).astype(bool)
    return out


def words_of(bits):
    """Inverse of bits_of: [n, 64*wq] bool -> [n*wq] uint64."""
    n, nb = bits.shape
    wq = nb // 64
    out = np.zeros((n, wq), dtype=U64)
    for w in range(wq):
        for b in range(64):
            out[:, w] |= bits[:, 64 * w + b].astype(U64) << U64(b)
    return out.reshape(-1)


def narrow_bits(D, n):
    D = np.asarray(D, dtype=U64)
    return np.array([[(int(D[x]) >> a) & 1 for a in range(64)] for x in range(n)], dtype=bool)


def duplicate(inst, k):
    """Every value a of x copied k times: copy j of a is value j*dom(x) + a of
    the wide instance; (a', b') allowed in c_xy iff (a' mod dom x, b' mod dom y)
    is allowed in the narrow c_xy.  Returns the wide Instance."""
    dom = np.asarray(inst.dom, dtype=np.int64)
    cons = []
    for r in range(inst.n_rel):
        x, y = int(inst.xs[r]), int(inst.ys[r])
        allowed = []
        for a in range(int(dom[x])):
            row = int(inst.rows[r, a])
            for b in range(int(dom[y])):
                if (row >> b) & 1:
                    for ja in range(k):
                        for jb in range(k):
                            allowed.append((ja * int(dom[x]) + a, jb * int(dom[y]) + b))
        cons.append((x, y, allowed))
    return synth.wide_from_constraints(inst.n, (dom * k).astype(np.int32), cons)


def duplicate_state(inst, k, D_narrow, rng=None):
    """A wide D_in over the duplicated instance.  Without rng every copy of a
    live value is live (the k-fold copy).  With rng each copy of a live value
    is kept at random (at least one copy of each live value stays), so copies
    of a value sit in different words with different liveness."""
    dom = np.asarray(inst.dom, dtype=np.int64)
    n = inst.n
    wq = synth.words_per_var(int(dom.max()) * k)
    nb = narrow_bits(D_narrow, n)
    wide = np.zeros((n, 64 * wq), dtype=bool)
    for x in range(n):
        for a in range(int(dom[x])):
            if not nb[x, a]:
                continue
            keep = np.ones(k, dtype=bool) if rng is None else rng.random(k) < 0.5
            if rng is not None and not keep.any():
                keep[rng.integers(k)] = True
            for j in range(k):
                if keep[j]:
                    wide[x, j * int(dom[x]) + a] = True
    return words_of(wide)


def project(inst, k, D_wide):
    """The narrow state whose values have at least one live copy."""
    dom = np.asarray(inst.dom, dtype=np.int64)
    n = inst.n
    wq = synth.words_per_var(int(dom.max()) * k)
    wb = bits_of(D_wide, n, wq)
    out = np.zeros(n, dtype=U64)
    for x in range(n):
        for a in range(int(dom[x])):
            if any(wb[x, j * int(dom[x]) + a] for j in range(k)):
                out[x] |= U64(1) << U64(a)
    return out


def restrict_domains(inst, dom):
    """The same instance with per-variable domain sizes dom[x] <= inst's: rows
    a >= dom[x] and columns b >= dom[y] of every relation dropped (input
    construction: no method arithmetic)."""
    dom = np.asarray(dom, dtype=np.int32)
    rows = np.array(inst.rows, dtype=U64, copy=True)
    nrel, dmax, wq = rows.shape
    for k in range(nrel):
        x, y = int(inst.xs[k]), int(inst.ys[k])
        rows[k, int(dom[x]):, :] = 0
        for w in range(wq):
            bits = min(64, max(0, int(dom[y]) - 64 * w))
            keep = U64(0xFFFFFFFFFFFFFFFF) if bits == 64 else U64((1 << bits) - 1)
            rows[k, :, w] &= keep
    return synth.Instance(n=inst.n, dom=dom, xs=inst.xs, ys=inst.ys, rows=rows)
