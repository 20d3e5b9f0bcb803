"""Seeded synthetic inputs for RAC: random binary CSPs and domain-state workloads.

INPUT GENERATION ONLY -- this module holds none of the method's arithmetic
(no support test, no recurrence, no arc-consistency check).  It is a numpy
port of ``synth/csp_synth.h`` (same frozen counter-based generator; the
specification is in that header and in DESIGN.md "Input recipe").  Both the
CPU oracle (``oracle/``) and the CUDA path are fed from here, as the task
rules permit; tests check that this port, the C header (used by the oracle)
and the device generator agree bit for bit.

Workload shapes follow PAPER.md §5.2 (lines 232-236): random binary CSPs
where each of the n(n-1)/2 pairs is constrained with probability = density.
Domain size and tightness are not stated by the paper; they are parameters
(SPEC.md instance_gen, lines 433-456).

Domain states use the C-ABI layout: one uint64 word per variable, bit a of
word x set iff value a is in D(x) (so dom sizes <= 64).
"""
from __future__ import annotations

import dataclasses
import json
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

U64 = np.uint64
M64 = (1 << 64) - 1

TAG_PRES = 0x50524553454E4345
TAG_CELL = 0x43454C4C42495453
TAG_KEEP = 0x4B454550424954
TAG_PICK = 0x5049434B43484F49
GAMMA = 0x9E3779B97F4A7C15


# ----------------------------------------------------------------------------- hashing
def mix64(z):
    """splitmix64 finalizer on a numpy uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=U64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> U64(30))
        z = z * U64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> U64(27))
        z = z * U64(0x94D049BB133111EB)
        z = z ^ (z >> U64(31))
    return z


def mix64_int(z: int) -> int:
    """Pure-int splitmix64 finalizer (scalar helper)."""
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def key(seed: int, tag: int) -> int:
    return mix64_int((seed & M64) ^ tag)


def quant_density(p: float) -> int:
    """density -> dens_q32 in [0, 2^32] (pair present iff hash>>32 < dens_q32)."""
    if not 0.0 <= p <= 1.0:
        raise ValueError("density must be in [0,1]")
    return int(round(p * (1 << 32)))


def quant_tightness(t: float) -> int:
    """tightness -> t_q16 in [0, 65536] (cell allowed iff 16-bit draw >= t_q16)."""
    if not 0.0 <= t <= 1.0:
        raise ValueError("tightness must be in [0,1]")
    return int(round(t * 65536))


def quant_keep(p: float) -> int:
    if not 0.0 <= p <= 1.0:
        raise ValueError("keep probability must be in [0,1]")
    return int(round(p * 65536))


# ----------------------------------------------------------------------------- instances
@dataclasses.dataclass
class Instance:
    """A binary CSP: n variables, per-variable domain sizes, one relation per
    constrained unordered pair stored in the x<y orientation.

    rows[k, a] is row a of rel(c_{xs[k] ys[k]}): bit b set iff (a,b) allowed
    (c_xy|(x,a) = {tau[y] | tau in rel(c_xy), tau[x] = a}).
    """

    n: int
    dom: np.ndarray  # int32 [n]
    xs: np.ndarray  # int32 [n_rel]
    ys: np.ndarray  # int32 [n_rel]
    rows: np.ndarray  # uint64 [n_rel, max_dom]
    gen: Optional[dict] = None

    @property
    def n_rel(self) -> int:
        return int(self.xs.shape[0])

    @property
    def max_dom(self) -> int:
        return int(self.dom.max()) if self.n else 0

    def full_domains(self) -> np.ndarray:
        return full_domains(self.dom)

    # SPEC.md csp_model "External Interfaces" (line 191): instance JSON format.
    def to_json(self) -> str:
        cons = []
        for k in range(self.n_rel):
            x, y = int(self.xs[k]), int(self.ys[k])
            allowed = []
            for a in range(int(self.dom[x])):
                r = int(self.rows[k, a])
                for b in range(int(self.dom[y])):
                    if (r >> b) & 1:
                        allowed.append([a, b])
            cons.append({"x": x, "y": y, "allowed": allowed})
        doc = {"n": self.n, "d": self.max_dom, "constraints": cons}
        if int(self.dom.min()) != int(self.dom.max()):
            doc["dom"] = [int(v) for v in self.dom]
        if self.gen is not None:
            doc["gen"] = self.gen
        return json.dumps(doc, sort_keys=True) + "\n"


def from_constraints(n: int, dom, constraints: Sequence[Tuple[int, int, Sequence[Tuple[int, int]]]],
                     gen: Optional[dict] = None) -> Instance:
    """Build an Instance from (x, y, allowed pairs) triples (x<y or x>y; stored x<y)."""
    if np.isscalar(dom):
        dom = [int(dom)] * n
    dom = np.asarray(dom, dtype=np.int32)
    dmax = int(dom.max()) if n else 1
    xs, ys, rows = [], [], []
    for (x, y, allowed) in constraints:
        if x > y:
            x, y = y, x
            allowed = [(b, a) for (a, b) in allowed]
        r = np.zeros(dmax, dtype=U64)
        for (a, b) in allowed:
            if not (0 <= a < dom[x] and 0 <= b < dom[y]):
                raise ValueError("value out of range")
            r[a] |= U64(1) << U64(b)
        xs.append(x)
        ys.append(y)
        rows.append(r)
    return Instance(n=n, dom=dom, xs=np.asarray(xs, dtype=np.int32), ys=np.asarray(ys, dtype=np.int32),
                    rows=np.asarray(rows, dtype=U64).reshape(len(rows), dmax), gen=gen)


def from_json(text: str) -> Instance:
    doc = json.loads(text)
    n = int(doc["n"])
    dom = doc.get("dom", [int(doc["d"])] * n)
    cons = [(c["x"], c["y"], [tuple(p) for p in c["allowed"]]) for c in doc["constraints"]]
    return from_constraints(n, dom, cons, gen=doc.get("gen"))


def present_pairs(n: int, dens_q32: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """All constrained pairs (x<y), ascending, per csp_synth.h synth_present."""
    x, y = np.triu_indices(n, k=1)
    x = x.astype(np.uint64)
    y = y.astype(np.uint64)
    kp = U64(key(seed, TAG_PRES))
    with np.errstate(over="ignore"):
        h = mix64(kp ^ mix64(x * U64(n) + y))
    keep = (h >> U64(32)) < U64(dens_q32) if dens_q32 < (1 << 32) else np.ones(h.shape, dtype=bool)
    return x[keep].astype(np.int32), y[keep].astype(np.int32)


def relation_rows(n: int, d: int, xs, ys, t_q16: int, seed: int) -> np.ndarray:
    """rows[k, a] for pairs (xs[k] < ys[k]) per csp_synth.h synth_row."""
    xs = np.asarray(xs, dtype=U64)
    ys = np.asarray(ys, dtype=U64)
    q = (d + 3) // 4
    kc = U64(key(seed, TAG_CELL))
    rows = np.zeros((xs.shape[0], d), dtype=U64)
    with np.errstate(over="ignore"):
        pk = mix64(kc ^ mix64(xs * U64(n) + ys))
        for a in range(d):
            acc = np.zeros(xs.shape[0], dtype=U64)
            for bq in range(q):
                h = mix64(pk + U64(a * q + bq + 1) * U64(GAMMA))
                for j in range(4):
                    b = bq * 4 + j
                    if b >= d:
                        break
                    v = (h >> U64(16 * j)) & U64(0xFFFF)
                    acc |= (v >= U64(t_q16)).astype(U64) << U64(b)
            rows[:, a] = acc
    return rows


def random_csp(n: int, d: int, density: float, tightness: float, seed: int) -> Instance:
    """Seeded random binary CSP (§5.2; generator spec in csp_synth.h)."""
    if not (1 <= d <= 64):
        raise ValueError("1 <= d <= 64")
    dq, tq = quant_density(density), quant_tightness(tightness)
    xs, ys = present_pairs(n, dq, seed)
    rows = relation_rows(n, d, xs, ys, tq, seed)
    return Instance(n=n, dom=np.full(n, d, dtype=np.int32), xs=xs, ys=ys, rows=rows,
                    gen={"n": n, "d": d, "density": density, "tightness": tightness,
                         "dens_q32": dq, "t_q16": tq, "seed": seed, "prng": "splitmix64-counter-v1"})


# ----------------------------------------------------------------------------- domain states
def full_domains(dom) -> np.ndarray:
    """W-root: every value present (the root call)."""
    dom = np.asarray(dom, dtype=np.int64)
    out = np.zeros(dom.shape[0], dtype=U64)
    for i, k in enumerate(dom):
        out[i] = U64((1 << int(k)) - 1) if k < 64 else U64(M64)
    return out


def w_rand(dom, keep: float, seed: int) -> np.ndarray:
    """W-rand: each value of the full domains kept with probability `keep` (seeded)."""
    dom = np.asarray(dom, dtype=np.int64)
    n = dom.shape[0]
    kq = U64(quant_keep(keep))
    kk = U64(key(seed, TAG_KEEP))
    out = np.zeros(n, dtype=U64)
    x = np.arange(n, dtype=U64)
    with np.errstate(over="ignore"):
        for a in range(int(dom.max()) if n else 0):
            h = mix64(kk ^ mix64(x * U64(64) + U64(a)))
            bit = ((h & U64(0xFFFF)) < kq) & (U64(a) < dom.astype(U64))
            out |= bit.astype(U64) << U64(a)
    return out


def pick(seed: int, k: int, m: int) -> int:
    """Seeded choice in [0, m)."""
    return mix64_int(key(seed, TAG_PICK) ^ mix64_int(k)) % m


def popcount64(v: int) -> int:
    return bin(int(v)).count("1")


def live_values(word: int) -> List[int]:
    w = int(word)
    return [a for a in range(64) if (w >> a) & 1]


def assign(D: np.ndarray, x: int, value: int) -> np.ndarray:
    """Alg. 2 `assign` as a row overwrite: D(x) := {value}."""
    out = np.array(D, dtype=U64, copy=True)
    out[x] = U64(1) << U64(value)
    return out


def w_seed(D_root: np.ndarray, seed: int, k: int = 0) -> Tuple[np.ndarray, int, int]:
    """W-seed: one seeded random variable of D_root assigned one seeded random live value
    (the paper's per-assignment unit)."""
    n = D_root.shape[0]
    cands = [x for x in range(n) if popcount64(D_root[x]) > 1]
    if not cands:
        cands = [x for x in range(n) if popcount64(D_root[x]) >= 1]
    x = cands[pick(seed, 2 * k, len(cands))]
    vals = live_values(D_root[x])
    v = vals[pick(seed, 2 * k + 1, len(vals))]
    return assign(D_root, x, v), x, v


def dive_states(D_root: np.ndarray, enforce: Callable[[np.ndarray], Tuple[int, np.ndarray]],
                n_states: int, seed: int, return_seeds: bool = False):
    """W-dive: chains of assignments (min-domain variable, lowest index tie-break,
    seeded random live value), each state being the input of one enforcement; restart
    from D_root after a wipeout or a complete assignment.  With return_seeds, also the
    assigned variable of each state (its Alg. 1 seed).  `enforce(D) -> (status, D_out)`
    is supplied by the caller (oracle in tests, the GPU path in bench), so this
    function holds none of the method's arithmetic."""
    states = []
    seeds = []
    cur = np.array(D_root, dtype=U64, copy=True)
    k = 0
    while len(states) < n_states:
        sizes = [popcount64(v) for v in cur]
        unassigned = [x for x in range(cur.shape[0]) if sizes[x] > 1]
        if not unassigned:
            cur = np.array(D_root, dtype=U64, copy=True)
            continue
        x = min(unassigned, key=lambda i: (sizes[i], i))
        vals = live_values(cur[x])
        v = vals[pick(seed, k, len(vals))]
        k += 1
        s = assign(cur, x, v)
        states.append(s)
        seeds.append(x)
        status, out = enforce(s)
        cur = np.array(D_root if status != 0 else out, dtype=U64, copy=True)
    return (states, seeds) if return_seeds else states


# ----------------------------------------------------------------------------- wide domains (NEXT-4)
# Domains of up to 256 values: a domain state is wq = ceil(dmax/64) uint64
# words per variable (bit a of x = bit a%64 of word x*wq + a//64), and
# Instance.rows becomes uint64 [n_rel, max_dom, wq].  Same generator spec as
# above (synth_allowed has no domain-size limit); input construction only.
def words_per_var(dmax: int) -> int:
    return max(1, (int(dmax) + 63) // 64)


def wide_from_constraints(n: int, dom, constraints, wq: Optional[int] = None) -> Instance:
    """Like from_constraints, rows as wq-word bitsets (wq defaults to ceil(max dom / 64))."""
    if np.isscalar(dom):
        dom = [int(dom)] * n
    dom = np.asarray(dom, dtype=np.int32)
    dmax = int(dom.max()) if n else 1
    wq = wq or words_per_var(dmax)
    xs, ys, rows = [], [], []
    for (x, y, allowed) in constraints:
        if x > y:
            x, y = y, x
            allowed = [(b, a) for (a, b) in allowed]
        r = np.zeros((dmax, wq), dtype=U64)
        for (a, b) in allowed:
            if not (0 <= a < dom[x] and 0 <= b < dom[y]):
                raise ValueError("value out of range")
            r[a, b >> 6] |= U64(1) << U64(b & 63)
        xs.append(x)
        ys.append(y)
        rows.append(r)
    return Instance(n=n, dom=dom, xs=np.asarray(xs, dtype=np.int32), ys=np.asarray(ys, dtype=np.int32),
                    rows=np.asarray(rows, dtype=U64).reshape(len(rows), dmax, wq))


def relation_rows_wide(n: int, d: int, xs, ys, t_q16: int, seed: int) -> np.ndarray:
    """rows[k, a, w] for pairs (xs[k] < ys[k]): csp_synth.h synth_allowed for any d."""
    xs = np.asarray(xs, dtype=U64)
    ys = np.asarray(ys, dtype=U64)
    q = (d + 3) // 4
    wq = words_per_var(d)
    kc = U64(key(seed, TAG_CELL))
    rows = np.zeros((xs.shape[0], d, wq), dtype=U64)
    with np.errstate(over="ignore"):
        pk = mix64(kc ^ mix64(xs * U64(n) + ys))
        for a in range(d):
            for bq in range(q):
                h = mix64(pk + U64(a * q + bq + 1) * U64(GAMMA))
                for j in range(4):
                    b = bq * 4 + j
                    if b >= d:
                        break
                    v = (h >> U64(16 * j)) & U64(0xFFFF)
                    rows[:, a, b >> 6] |= (v >= U64(t_q16)).astype(U64) << U64(b & 63)
    return rows


def random_csp_wide(n: int, d: int, density: float, tightness: float, seed: int) -> Instance:
    """The seeded random instance of csp_synth.h for 1 <= d <= 256 (rows [n_rel, d, wq])."""
    if not (1 <= d <= 256):
        raise ValueError("1 <= d <= 256")
    dq, tq = quant_density(density), quant_tightness(tightness)
    xs, ys = present_pairs(n, dq, seed)
    rows = relation_rows_wide(n, d, xs, ys, tq, seed)
    return Instance(n=n, dom=np.full(n, d, dtype=np.int32), xs=xs, ys=ys, rows=rows,
                    gen={"n": n, "d": d, "density": density, "tightness": tightness,
                         "dens_q32": dq, "t_q16": tq, "seed": seed, "prng": "splitmix64-counter-v1"})


def full_domains_wide(dom, wq: Optional[int] = None) -> np.ndarray:
    """W-root on wide domains: [n * wq] words, every value of dom(x) present."""
    dom = np.asarray(dom, dtype=np.int64)
    wq = wq or words_per_var(int(dom.max()) if dom.size else 1)
    out = np.zeros((dom.shape[0], wq), dtype=U64)
    for i, k in enumerate(dom):
        for w in range(wq):
            bits = min(64, max(0, int(k) - 64 * w))
            out[i, w] = U64(M64) if bits == 64 else U64((1 << bits) - 1)
    return out.reshape(-1)


def w_rand_wide(dom, keep: float, seed: int, wq: Optional[int] = None) -> np.ndarray:
    """W-rand on wide domains: value (x,a) kept with probability `keep`, hashed on x*256 + a."""
    dom = np.asarray(dom, dtype=np.int64)
    n = dom.shape[0]
    wq = wq or words_per_var(int(dom.max()) if n else 1)
    kq = U64(quant_keep(keep))
    kk = U64(key(seed, TAG_KEEP))
    out = np.zeros((n, wq), dtype=U64)
    x = np.arange(n, dtype=U64)
    with np.errstate(over="ignore"):
        for a in range(int(dom.max()) if n else 0):
            h = mix64(kk ^ mix64(x * U64(256) + U64(a)))
            bit = ((h & U64(0xFFFF)) < kq) & (U64(a) < dom.astype(U64))
            out[:, a >> 6] |= bit.astype(U64) << U64(a & 63)
    return out.reshape(-1)
