"""Synthetic labeled streams as flat arrays -- TEST INFRASTRUCTURE ONLY.

numpy restatement of the reference generator `simharness.generate_stream`
(/root/reference/pkg/src/focusidx/simharness.py:32-156), drawing the same
numpy Generator calls in the same order so that, for the same StreamSpec,
the arrays are bit-identical to the reference's DetectedObject fields
(checked by tools/gen_golden.py, which stores input digests that
tests/test_oracle.py re-verifies).  Returned as arrays because the GPU path
and the oracle both consume arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_PIXEL_EPS = 0.01  # ingest.py:23


@dataclass(frozen=True)
class Spec:
    """Field-for-field the reference StreamSpec (simharness.py:32-47)."""
    n_objects: int = 10_000
    fps: float = 30.0
    vocab: int = 1000
    n_stream_classes: int = 100
    zipf_s: float = 2.5
    duplicate_rate: float = 0.2
    objects_per_frame: float = 1.0
    segment_class_slots: int = 3
    rare_visitor_rate: float = 0.5
    dim: int = 64
    sig_dim: int = 16
    class_sigma: float = 0.1
    seed: int = 0
    stream_id: str = "synthetic"


@dataclass
class Stream:
    spec: Spec
    oids: np.ndarray        # int64[n]
    fids: np.ndarray        # int64[n]
    sigs: np.ndarray        # float64[n, sig_dim]
    feats: np.ndarray       # float64[n, dim]  (pre-extraction feature)
    true_class: np.ndarray  # int64[n]


def _schedule(rng, spec: Spec, weights, n_base):
    """(frame, class-index) of the non-duplicate detections (simharness.py:100-128)."""
    frames, cis = [], []
    seg = max(1, int(round(spec.fps)))
    frame, active, shares = 0, None, None
    visitor_left = visitor = 0
    while len(frames) < n_base:
        if active is None or frame % seg == 0:
            active = rng.choice(spec.n_stream_classes, size=spec.segment_class_slots, p=weights)
            shares = rng.dirichlet(np.ones(spec.segment_class_slots))
            if rng.random() < spec.rare_visitor_rate:
                visitor = int(rng.integers(spec.n_stream_classes))
                visitor_left = 2
        for _ in range(rng.poisson(spec.objects_per_frame)):
            frames.append(frame)
            cis.append(int(rng.choice(active, p=shares)))
        if visitor_left:
            frames.append(frame)
            cis.append(visitor)
            visitor_left -= 1
        frame += 1
    return frames[:n_base], cis[:n_base]


def generate(spec: Spec) -> Stream:
    n = spec.n_objects
    oids = np.arange(n, dtype=np.int64)
    fids = np.zeros(n, dtype=np.int64)
    sigs = np.zeros((n, spec.sig_dim))
    feats = np.zeros((n, spec.dim))
    tcls = np.zeros(n, dtype=np.int64)
    if n == 0:
        return Stream(spec, oids, fids, sigs, feats, tcls)
    rng = np.random.default_rng([spec.seed, 0xA110])
    classes = rng.choice(spec.vocab, size=spec.n_stream_classes, replace=False)
    w = np.arange(1, spec.n_stream_classes + 1, dtype=float) ** -spec.zipf_s
    w /= w.sum()
    means = rng.standard_normal((spec.n_stream_classes, spec.dim))
    n_dup = int(round(spec.duplicate_rate * n)) if n > 1 else 0
    dup_at = np.zeros(n, dtype=bool)
    if n_dup:
        dup_at[rng.choice(n - 1, size=n_dup, replace=False) + 1] = True
    frames, cis = _schedule(rng, spec, w, n - n_dup)
    eps = DEFAULT_PIXEL_EPS
    j = 0
    for pos in range(n):
        if dup_at[pos]:
            sigs[pos] = sigs[pos - 1] + rng.uniform(-eps / 4, eps / 4, spec.sig_dim)
            feats[pos] = feats[pos - 1] + 0.01 * rng.standard_normal(spec.dim)
            fids[pos] = fids[pos - 1]
            tcls[pos] = tcls[pos - 1]
        else:
            ci = cis[j]
            fids[pos] = frames[j]
            j += 1
            feats[pos] = means[ci] + spec.class_sigma * rng.standard_normal(spec.dim)
            s = rng.standard_normal(spec.sig_dim)
            s[0] = float(pos)
            sigs[pos] = s
            tcls[pos] = int(classes[ci])
    return Stream(spec, oids, fids, sigs, feats, tcls)
