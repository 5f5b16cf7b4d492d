"""Helpers to read tests/golden/golden.json and hash arrays like the generator."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")


def h(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()[:32]


def load_cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["cases"]


def case_inputs(case):
    """(costs, rows, chunk) of a golden case; product-space rows are rebuilt."""
    from tests.cases import csr_hash, product_space

    if "config" in case:
        p = product_space(case["config"], case.get("seed", 0))
        assert csr_hash(p) == case["rows_hash"], "product-space builder output changed"
        return p.costs, p, case["chunk"]
    rows = [(np.asarray(v, np.int64), np.asarray(c, np.int64), int(b)) for v, c, b in case["rows"]]
    return np.asarray(case["costs"], np.float64), rows, case["chunk"]


FLAT_FIELDS = ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t", "one_t", "proc_ptr",
               "proc_layers")


PRIMAL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "primal.json")


def load_primal_cases():
    with open(PRIMAL) as fh:
        return json.load(fh)["cases"]
