"""Device-side synthetic streams for benchmarking.

Same statistical model as the reference generator (simharness.py:74-156):
per-stream class means ~ N(0, I); a Zipf(2.5) class mix over
n_stream_classes classes drawn from the vocabulary; exactly
round(duplicate_rate * n) near-duplicate detections (same frame, pixel
signature within eps/4 of the predecessor); every other adjacent pair differs
by more than eps (signature coordinate 0 carries the emission counter).  The
feature the ingest clusters is the cheap CNN's output: class mean +
sqrt(class_sigma^2 + noise_sigma^2) * N(0, I), in float32.  A 10M x 2048
float64 stream does not fit host RAM, so benchmarks generate on the device
(torch is plumbing here); parity is checked on reference-generated prefixes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SynthStream:
    n: int
    dim: int
    sig_dim: int
    vocab: int
    oids: "object"        # torch int64 [n]
    fids: "object"        # torch int64 [n]
    sigs: "object"        # torch float64 [n, S]
    feats: "object"       # torch float32 [n, D]
    true_class: "object"  # torch int32 [n]
    is_dup: "object"      # torch bool [n] (intended duplicates)


def generate(n: int, dim: int = 2048, vocab: int = 1000, n_stream_classes: int = 100, seed: int = 0,
             zipf_s: float = 2.5, duplicate_rate: float = 0.2, class_sigma: float = 0.1, noise_sigma: float = 0.05,
             sig_dim: int = 16, device="cuda") -> SynthStream:
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(0x5EED0000 + seed)
    hg = np.random.default_rng([seed, 0xB200])
    classes = torch.from_numpy(hg.choice(vocab, size=n_stream_classes, replace=False).astype(np.int32)).to(device)
    w = np.arange(1, n_stream_classes + 1, dtype=np.float64) ** -zipf_s
    w /= w.sum()
    means = torch.randn(n_stream_classes, dim, generator=g, device=device, dtype=torch.float32)
    n_dup = int(round(duplicate_rate * n)) if n > 1 else 0
    is_dup = torch.zeros(n, dtype=torch.bool, device=device)
    if n_dup:
        pos = torch.from_numpy(hg.choice(n - 1, size=n_dup, replace=False) + 1).to(device)
        is_dup[pos] = True
    ci = torch.multinomial(torch.from_numpy(w).to(device), n, replacement=True, generator=g)
    # duplicates inherit their predecessor's class / frame / features
    idx = torch.arange(n, device=device)
    anchor = torch.where(~is_dup, idx, torch.zeros_like(idx))
    anchor = torch.cummax(anchor, 0).values
    ci = ci[anchor]
    sig_eff = float(np.sqrt(class_sigma ** 2 + noise_sigma ** 2))
    feats = torch.empty(n, dim, dtype=torch.float32, device=device)
    chunk = 1 << 16
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        feats[a:b] = means[ci[a:b]] + sig_eff * torch.randn(b - a, dim, generator=g, device=device)
    sigs = torch.randn(n, sig_dim, generator=g, device=device, dtype=torch.float64)
    sigs[:, 0] = idx.to(torch.float64)
    eps = 0.01
    jitter = (torch.rand(n, sig_dim, generator=g, device=device, dtype=torch.float64) - 0.5) * (eps / 2)
    sigs = torch.where(is_dup[:, None], sigs[anchor] + jitter, sigs)
    # frames: each non-duplicate detection opens the next frame; duplicates share it
    fids = torch.cumsum((~is_dup).to(torch.int64), 0) - 1
    return SynthStream(n=n, dim=dim, sig_dim=sig_dim, vocab=vocab, oids=idx.to(torch.int64), fids=fids,
                       sigs=sigs.contiguous(), feats=feats, true_class=classes[ci].to(torch.int32),
                       is_dup=is_dup)
