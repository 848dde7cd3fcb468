"""Oracle restatement of the inference half of the reference predictor.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Follows
/root/reference/pkg/src/moesim/predictor.py: feature layout (:49-51,
:81-128), flat-node tree walk (:225-232), forest mean / residual (:327-349),
JSON format ``moesim-forest`` v1 (:575-632), and the embedding table of
workload.py:31-45.
"""

from __future__ import annotations

import json
from typing import Dict, Mapping, Sequence, Tuple

import numpy as np

from .decisions import seed_split  # noqa: F401  (re-exported for tests)


def embedding_table(vocab: int, dim: int, seed_value: int) -> np.ndarray:
    """workload.py:41-45 — U[-1, 1] from PCG64(seed)."""
    return np.random.default_rng(seed_value).uniform(-1.0, 1.0, size=(vocab, dim))


def pooled(table: np.ndarray, token_ids: Sequence[int]) -> np.ndarray:
    """predictor.py:76-78 — row mean (sequential row sum / n)."""
    acc = np.zeros(table.shape[1], dtype=np.float64)
    for t in token_ids:
        acc = acc + table[t]
    return acc / len(token_ids)


def history_bits(L: int, M: int, history: Mapping[int, Tuple[int, ...]], below: int) -> np.ndarray:
    """predictor.py:81-100 — slot k holds layer below-1-k."""
    bits = np.zeros(L * M, dtype=np.float64)
    for layer, experts in history.items():
        if 0 <= layer < below and below - 1 - layer < L:
            for e in experts:
                bits[(below - 1 - layer) * M + e] = 1.0
    return bits


def features(table, L, M, token_ids, step, target, history) -> np.ndarray:
    """predictor.py:113-128."""
    return np.concatenate((pooled(table, token_ids), [float(step), float(target)],
                           history_bits(L, M, history, target)))


class Forest:
    """predictor.py:293-349 over flat node arrays."""

    def __init__(self, payload: dict):
        if payload.get("format") != "moesim-forest" or payload.get("version") != 1:
            raise ValueError("not a moesim-forest v1 payload")
        self.residual = bool(payload["hyper"]["residual"])
        self.feature_len = int(payload["feature_len"])
        self.num_outputs = int(payload["num_outputs"])
        self.trees = payload["trees"]

    @classmethod
    def from_json(cls, text: str) -> "Forest":
        return cls(json.loads(text))

    def _leaf(self, tree, x):
        n = 0
        while tree["feature"][n] != -1:
            n = tree["left"][n] if x[tree["feature"][n]] <= tree["threshold"][n] else tree["right"][n]
        return np.asarray(tree["value"][n], dtype=np.float64)

    def predict_scores(self, x, baseline=None) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.feature_len,):
            raise ValueError("wrong feature length")
        acc = np.zeros(self.num_outputs, dtype=np.float64)
        for tree in self.trees:
            acc += self._leaf(tree, x)
        acc /= len(self.trees)
        if self.residual:
            if baseline is None:
                raise ValueError("residual model needs a baseline distribution")
            return np.asarray(baseline, dtype=np.float64) + acc
        return acc
