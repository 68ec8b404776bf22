"""Stream-sharded deployment.

Streams are independent (one engine per stream, clustering.py:87; "cross-
stream parallelism ... process-level"), so stream s lives on
rank s % world and ingest needs no inter-GPU traffic.  A query touches every
stream: each rank runs K4/K5 on its own streams and the per-stream results
are merged with two all-gathers (counts, then payloads padded to the largest
count) -- over NCCL / NVLink when the process group is NCCL, with the id
lists never leaving device memory; over gloo (CPU tensors) otherwise.
Concatenating the gathered blocks in rank order and placing them by stream
index gives every rank the full result in stream order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_HDR = 6  # stream index, n_frames, n_objects, gt_inferences, clusters_examined, clusters_matched


def owner(stream_index: int, world: int) -> int:
    """Rank that ingests and queries stream `stream_index`."""
    return stream_index % world


def local_streams(n_streams: int, rank: int, world: int) -> list:
    return [s for s in range(n_streams) if owner(s, world) == rank]


@dataclass
class StreamResult:
    """One stream's part of a sharded query (ids as int64 arrays)."""
    stream_index: int
    frame_ids: np.ndarray
    object_ids: np.ndarray
    gt_inferences: int
    clusters_examined: int
    clusters_matched: int


def _torch():
    import torch
    import torch.distributed as dist
    return torch, dist


def _pack(torch, parts, device):
    """parts: list of (stream_index, frames_tensor, objects_tensor, stats) -> one int64 tensor."""
    n = len(parts)
    hdr = torch.empty(1 + _HDR * n, dtype=torch.int64)
    hdr[0] = n
    for i, (si, fr, ob, st) in enumerate(parts):
        hdr[1 + _HDR * i: 1 + _HDR * (i + 1)] = torch.tensor([si, fr.numel(), ob.numel(), *st], dtype=torch.int64)
    pieces = [hdr.to(device)]
    for _, fr, ob, _ in parts:
        pieces += [fr.to(device), ob.to(device)]
    return torch.cat(pieces)


def merge(parts, n_streams: int, group=None) -> list:
    """All-gather the local streams' results of one query.

    parts: list of (stream_index, frame_ids, object_ids, (gt, examined, matched))
    with the id lists as torch int64 tensors (CUDA tensors for an NCCL group)
    or numpy arrays.  Returns a list of StreamResult indexed by stream."""
    torch, dist = _torch()
    nccl = dist.get_backend(group) == "nccl"
    device = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    tparts = []
    for si, fr, ob, st in parts:
        fr = torch.as_tensor(fr, dtype=torch.int64)
        ob = torch.as_tensor(ob, dtype=torch.int64)
        tparts.append((si, fr, ob, st))
    payload = _pack(torch, tparts, device)
    world = dist.get_world_size(group)
    size = torch.tensor([payload.numel()], dtype=torch.int64, device=device)
    sizes = [torch.empty_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    buf = torch.zeros(mx, dtype=torch.int64, device=device)
    buf[:payload.numel()] = payload
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    out = [None] * n_streams
    for r in range(world):
        b = bufs[r][:sizes[r]].cpu().numpy()
        n = int(b[0])
        hdr = b[1:1 + _HDR * n].reshape(n, _HDR)
        off = 1 + _HDR * n
        for si, nf, no, gt, ex, ma in hdr.tolist():
            fr = b[off:off + nf]
            ob = b[off + nf:off + nf + no]
            off += nf + no
            out[si] = StreamResult(si, fr.copy(), ob.copy(), gt, ex, ma)
    return out


class ShardedQuery:
    """Queries over stream-sharded indexes.  `sessions` maps this rank's stream
    indexes to their QuerySession (query.py); every rank calls `query` with
    the same request (the descriptor is replicated)."""

    def __init__(self, sessions: dict, n_streams: int, group=None):
        self.sessions = dict(sessions)
        self.n_streams = n_streams
        self.group = group

    def query(self, req, fresh: bool = True) -> list:
        torch, dist = _torch()
        nccl = dist.get_backend(self.group) == "nccl"
        parts = []
        for si in sorted(self.sessions):
            s = self.sessions[si]
            if fresh:
                s.reset()
            if nccl:
                # ids stay in HBM: sized by the query, copied device-to-device
                nf, no, st = s.query_device(req)
                fr = torch.empty(nf, dtype=torch.int64, device="cuda")
                ob = torch.empty(no, dtype=torch.int64, device="cuda")
                if nf or no:
                    s.fetch_device(fr, ob)
                parts.append((si, fr, ob, st))
            else:
                fr, ob, st = s.query_arrays(req)
                parts.append((si, fr, ob, st))
        return merge(parts, self.n_streams, self.group)
