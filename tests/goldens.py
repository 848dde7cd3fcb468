"""Loaders for the golden fixtures in tests/golden/ (made by make_golden.py
from the real reference).  Shared by the oracle tests and the product tests."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name: str):
    with open(os.path.join(GOLDEN_DIR, name)) as f:
        return json.load(f)


def token_trace(tj):
    from oracle.sim import TokenTrace
    return TokenTrace(
        token_ids=tuple(tj["token_ids"]),
        gates=[np.asarray(g, dtype=np.float64) for g in tj["gates"]],
        actual=[tuple(a) for a in tj["actual"]],
        group_actual=[tuple(tuple(g) for g in layer) for layer in tj["group_actual"]],
        group_sizes=tuple(tj["group_sizes"]),
    )


def oracle_policy(pj):
    from oracle.sim import Policy
    return Policy(**pj)


def seconds_to_ns(s):
    return round(s * 1_000_000_000)
