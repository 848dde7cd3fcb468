"""Inference half of the hybrid predictor: feature rows and forest scoring in
the C++ runtime (reference predictor.py:49-51, :81-128, :195-232, :293-359,
:575-632).  Training and accuracy analysis are offline tooling and stay out
of this package; ``moesim-forest`` v1 JSON files trained by the
reference load unchanged."""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Mapping, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .core import ModelSpec
from .workload import EmbeddingTable


def feature_length(model: ModelSpec) -> int:
    """F = embed_dim + 2 + num_layers * experts_per_layer."""
    return model.embed_dim + 2 + model.num_layers * model.experts_per_layer


def _hist(history: Mapping[int, Tuple[int, ...]]) -> Tuple[np.ndarray, int]:
    rec = []
    for layer, ex in history.items():
        rec += [int(layer), len(ex), *map(int, ex)]
    return L.i32arr(rec or [0]), len(rec)


def inference_features(model: ModelSpec, table: EmbeddingTable, token_ids: Tuple[int, ...],
                       step: int, target_layer: int,
                       history: Mapping[int, Tuple[int, ...]]) -> np.ndarray:
    vec = L.f64arr(table.vectors)
    toks = L.i64arr(list(token_ids) or [0])
    hist, n = _hist(history)
    out = np.empty(feature_length(model), dtype=np.float64)
    L.check(L.lib.ef_inference_features(
        L.as_ptr(vec, C.c_double), vec.shape[0], vec.shape[1], model.num_layers,
        model.experts_per_layer, L.as_ptr(toks, C.c_int64), len(token_ids), int(step),
        int(target_layer), L.as_ptr(hist, C.c_int32), n, L.as_ptr(out, C.c_double)))
    return out


@dataclass(frozen=True)
class ForestHyper:
    num_trees: int = 50
    max_depth: int = 12
    min_samples_leaf: int = 2
    residual: bool = False

    def __post_init__(self) -> None:
        if self.num_trees < 1:
            raise ValueError(f"num_trees must be >= 1, got {self.num_trees}")
        if self.max_depth < 1:
            raise ValueError(f"max_depth must be >= 1, got {self.max_depth}")
        if self.min_samples_leaf < 1:
            raise ValueError(f"min_samples_leaf must be >= 1, got {self.min_samples_leaf}")


@dataclass
class _Tree:
    """Flat node arrays; feature == -1 marks a leaf (predictor.py:183-232)."""
    feature: List[int] = field(default_factory=list)
    threshold: List[float] = field(default_factory=list)
    left: List[int] = field(default_factory=list)
    right: List[int] = field(default_factory=list)
    value: List[Optional[List[float]]] = field(default_factory=list)


@dataclass
class ForestModel:
    trees: List[_Tree]
    hyper: ForestHyper
    train_seed: int
    feature_len: int
    num_outputs: int
    embedding_seed: Optional[int] = None

    def _native_handle(self):
        h = getattr(self, "_native", None)
        if h is None:
            off = [0]
            feat, thr, lft, rgt, val = [], [], [], [], []
            for t in self.trees:
                feat += t.feature
                thr += t.threshold
                lft += t.left
                rgt += t.right
                for v in t.value:
                    val += (v if v is not None else [0.0] * self.num_outputs)
                off.append(len(feat))
            arrs = dict(off=L.i64arr(off), feat=L.i32arr(feat), thr=L.f64arr(thr),
                        lft=L.i32arr(lft), rgt=L.i32arr(rgt), val=L.f64arr(val))
            ptr = L.vp()
            L.check(L.lib.ef_forest_create(
                len(self.trees), L.as_ptr(arrs["off"], C.c_int64), L.as_ptr(arrs["feat"], C.c_int32),
                L.as_ptr(arrs["thr"], C.c_double), L.as_ptr(arrs["lft"], C.c_int32),
                L.as_ptr(arrs["rgt"], C.c_int32), L.as_ptr(arrs["val"], C.c_double),
                self.feature_len, self.num_outputs, int(self.hyper.residual), C.byref(ptr)))
            h = L.Handle(ptr.value, L.lib.ef_forest_destroy)
            object.__setattr__(self, "_native", h)
        return h.ptr

    def predict_scores(self, features: np.ndarray,
                       baseline: Optional[np.ndarray] = None) -> np.ndarray:
        x = L.f64arr(features)
        if x.shape != (self.feature_len,):
            raise ValueError(f"expected feature vector of length {self.feature_len}, "
                             f"got shape {x.shape}")
        out = np.empty(self.num_outputs, dtype=np.float64)
        base = None
        if baseline is not None:
            base = L.f64arr(baseline)
        L.check(L.lib.ef_forest_predict(self._native_handle(), L.as_ptr(x, C.c_double),
                                        None if base is None else L.as_ptr(base, C.c_double),
                                        L.as_ptr(out, C.c_double)))
        return out

    def predict_matrix(self, X: np.ndarray, baselines: Optional[np.ndarray] = None) -> np.ndarray:
        X = np.asarray(X, dtype=np.float64)
        return np.stack([self.predict_scores(X[i], None if baselines is None else baselines[i])
                         for i in range(X.shape[0])]) if len(X) else \
            np.empty((0, self.num_outputs))


def model_to_json(model: ForestModel) -> str:
    payload = {
        "format": "moesim-forest", "version": 1,
        "hyper": {"num_trees": model.hyper.num_trees, "max_depth": model.hyper.max_depth,
                  "min_samples_leaf": model.hyper.min_samples_leaf,
                  "residual": model.hyper.residual},
        "train_seed": model.train_seed, "feature_len": model.feature_len,
        "num_outputs": model.num_outputs, "embedding_seed": model.embedding_seed,
        "trees": [{"feature": t.feature, "threshold": t.threshold, "left": t.left,
                   "right": t.right, "value": t.value} for t in model.trees],
    }
    return json.dumps(payload, sort_keys=True, separators=(",", ":"))


def model_from_json(text: str) -> ForestModel:
    d = json.loads(text)
    if d.get("format") != "moesim-forest":
        raise ValueError(f"not a forest file: format={d.get('format')!r}")
    if d.get("version") != 1:
        raise ValueError(f"unsupported forest version {d.get('version')!r}")
    trees = [_Tree(list(t["feature"]), [float(v) for v in t["threshold"]], list(t["left"]),
                   list(t["right"]),
                   [None if v is None else [float(x) for x in v] for v in t["value"]])
             for t in d["trees"]]
    return ForestModel(trees, ForestHyper(**d["hyper"]), d["train_seed"], d["feature_len"],
                       d["num_outputs"], d.get("embedding_seed"))
