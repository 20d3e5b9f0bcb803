"""Structured test instances with closed-form answers, and random tiny corpora.

Test-only helpers (constructors of inputs, no method arithmetic).
"""
from __future__ import annotations

import json
import os

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        doc = json.load(f)
    inst = synth.from_json(json.dumps(doc["instance"]))
    return doc, inst


def golden_names():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".json"))


def eq_rel(d):
    return [(a, a) for a in range(d)]


def equality_chain(n, d, embed_complete=False):
    """x_i = x_{i+1} for i < n-1.  With embed_complete, every other pair carries a
    present all-ones relation (complete constraint graph)."""
    cons = [(i, i + 1, eq_rel(d)) for i in range(n - 1)]
    if embed_complete:
        allp = [(a, b) for a in range(d) for b in range(d)]
        for x in range(n):
            for y in range(x + 2, n):
                cons.append((x, y, allp))
    return synth.from_constraints(n, d, cons)


def random_corpus(count, seed0=1, n_range=(2, 20), d_range=(1, 6), dens=(0.1, 1.0), tight=(0.0, 0.9)):
    """SPEC.md acceptance corpus shape (line 528): n in 2..20, d in 1..6,
    density 0.1..1.0, tightness 0..0.9, seeded deterministically."""
    rng = np.random.default_rng(seed0)
    out = []
    for i in range(count):
        n = int(rng.integers(n_range[0], n_range[1] + 1))
        d = int(rng.integers(d_range[0], d_range[1] + 1))
        p = float(rng.uniform(*dens))
        t = float(rng.uniform(*tight))
        out.append(synth.random_csp(n, d, p, t, seed=seed0 * 100003 + i))
    return out


def tiny_corpus(count, seed0=7):
    """Instances small enough for brute force: n <= 5, d <= 4, n*d <= 14."""
    rng = np.random.default_rng(seed0)
    out = []
    while len(out) < count:
        n = int(rng.integers(1, 6))
        d = int(rng.integers(1, 5))
        if n * d > 14:
            continue
        p = float(rng.uniform(0.2, 1.0))
        t = float(rng.uniform(0.0, 0.8))
        out.append(synth.random_csp(n, d, p, t, seed=seed0 * 7919 + len(out)))
    return out
