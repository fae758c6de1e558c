"""Host-side data-parallel partitioning of the model points.

Rank r of a world of N owns the points whose primary node (smallest node id of
their kNN tuple) falls in its node-row range; the ranges are contiguous and
balanced by point count, so a rank's points are spatially coherent (node ids
follow the node grid) and the per-rank block systems overlap only on the node
rows at range boundaries.  Each rank passes its shard to mis_set_model /
mis_set_graph with *global* node ids; the library all-reduces the point-term
accumulators and energies (they are linear in the per-rank sums); the
regulariser and feature terms are computed by every rank alike and not reduced.
"""
from __future__ import annotations

import numpy as np


def node_ranges(primary: np.ndarray, m: int, world: int) -> np.ndarray:
    """Boundaries b[0..world] over node ids so that each range holds ~n/world points."""
    counts = np.bincount(primary, minlength=m)
    cum = np.concatenate([[0], np.cumsum(counts)])
    n = cum[-1]
    b = np.searchsorted(cum, [n * r / world for r in range(world + 1)], side="left")
    b[0], b[-1] = 0, m
    return np.maximum.accumulate(b)


def shard_indices(knn_idx: np.ndarray, m: int, world: int, rank: int) -> np.ndarray:
    """Indices of the points rank `rank` owns (disjoint over ranks, covering all points)."""
    primary = np.asarray(knn_idx).min(axis=1)
    b = node_ranges(primary, m, world)
    return np.flatnonzero((primary >= b[rank]) & (primary < b[rank + 1]))


def graph_terms_on(rank: int) -> bool:
    """In a sum of per-shard systems (P15) the regulariser (Eq. 6) and feature (Eq. 9) terms count
    once: shard 0 carries them.  (libmis itself computes them on every rank and reduces only the
    point terms, which gives the same total.)"""
    return rank == 0
