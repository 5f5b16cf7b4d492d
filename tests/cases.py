"""Deterministic test instances shared by the golden generator and the tests."""

from __future__ import annotations

import hashlib

import numpy as np

from paper_2310_08230_b200 import product_space as ps


def random_rows(seed: int, num_vars: int = 14, num_rows: int = 6):
    """Random feasible 0-1 equality rows (reference test style, test_qn.py:160-170)."""
    rng = np.random.default_rng(seed)
    rows = []
    attempts = 0
    while len(rows) < num_rows and attempts < 50 * num_rows:
        attempts += 1
        k = int(rng.integers(2, min(6, num_vars) + 1))
        v = np.sort(rng.choice(num_vars, size=k, replace=False))
        c = rng.integers(-2, 3, size=k)
        if not c.any():
            continue
        bits = rng.integers(0, 2, size=k)
        rows.append((v, c, int(c @ bits)))
    costs = rng.standard_normal(num_vars) * 2.0
    return costs, rows


def csr_hash(p: ps.ProductSpace) -> str:
    m = hashlib.sha256()
    for a in (p.row_ptr, p.row_var, p.row_coef, p.row_rhs, p.costs):
        a = np.ascontiguousarray(a)
        m.update(a.dtype.str.encode() + a.tobytes())
    return m.hexdigest()[:32]


def product_space(cfg: str, seed: int = 0) -> ps.ProductSpace:
    return ps.synthetic_product_space(cfg, seed)


def product_case(cfg: str, seed: int = 0):
    p = product_space(cfg, seed)
    return p.costs, p.rows(), {"config": cfg, "seed": seed, "rows_hash": csr_hash(p)}
