"""Cluster records (drop-in for focusidx.clustering.Cluster).

The clustering engine itself (clustering.py:86-160) is the device pipeline in
csrc/ingest.cu, driven through ingest.ingest_stream / ingest_arrays; this
module keeps the record type the index and callers exchange.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._reftypes import shared


@dataclass
class Cluster:
    cluster_id: int
    centroid: np.ndarray
    member_object_ids: list = field(default_factory=list)
    frame_ids: list = field(default_factory=list)
    class_best_rank: dict = field(default_factory=dict)
    centroid_member_id: int | None = None
    sealed: bool = False
    insertion_distances: list = field(default_factory=list)

    @property
    def class_set(self) -> set:
        return set(self.class_best_rank)

    def size(self) -> int:
        return len(self.member_object_ids)


Cluster = shared("clustering", "Cluster", Cluster)
