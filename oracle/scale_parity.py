"""At-scale parity check -- TEST INFRASTRUCTURE ONLY.

Runs the device ingest (libfocus_b200.so through the product package) and
the CPU oracle (oracle.py / focus_oracle.c, the reference algorithm restated:
ingest.py:50-96, clustering.py:104-153, index.py:60-72) on the SAME stream and
compares every output bit for bit:

  is_dup (ingest.py:37-47, 69-71), top-K of classified objects
  (classifiers.py:136-149), cluster of every object (clustering.py:104-132),
  distance_computations (clustering.py:117), float64 centroid bits
  (clustering.py:56-59), representatives (clustering.py:71-83), member and
  frame lists (clustering.py:49-63), class best ranks (clustering.py:65-69),
  postings (index.py:60-72).

Used by tests/test_gpu_scale_parity.py and by ``bench.py`` (the ``parity``
key of its JSON line; run after the timed region, never inside it).  The
stream is the bench's own device-generated stream (synth.generate) copied to
the host, so the check covers exactly the objects the headline number is
quoted on.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import oracle as O


def device_ingest(data, n: int, k: int, t: float, m: int, vocab: int, profile, seed: int = 0,
                  device: int = 0, batch: int = 0) -> dict:
    """Ingest the first n objects of a synth stream (torch tensors on the
    device) through the C ABI and export everything the check compares."""
    import paper_1801_03493_b200 as fx
    from paper_1801_03493_b200 import _lib
    s = fx.ingest.Stream(data.dim, data.sig_dim, vocab, k, t, m, 0.01, _lib.FX_F32, device, batch)
    s.set_rank_model(profile, seed)
    s.ingest_device(n, data.oids.data_ptr(), data.fids.data_ptr(), data.sigs.data_ptr(), data.feats.data_ptr(),
                    data.true_class.data_ptr())
    dix, rep = s.finalize()
    cl, dup, tk = s.object_results(n, k)
    out = dict(cluster_of=cl.astype(np.int64), is_dup=dup, topk=tk, dc=int(rep.distance_computations),
               exact_rechecks=int(rep.exact_rechecks), counters=s.counters())
    out.update(dix.export(centroids=True))
    del dix, s
    return out


def host_stream(data, n: int) -> dict:
    """The first n objects of a device synth stream as host arrays."""
    return dict(oids=data.oids[:n].cpu().numpy(), fids=data.fids[:n].cpu().numpy(),
                sigs=data.sigs[:n].cpu().numpy(), feats=data.feats[:n].cpu().numpy(),
                true_class=data.true_class[:n].cpu().numpy())


def oracle_ingest(h: dict, k: int, t: float, m: int, vocab: int, seed: int = 0, threads: int | None = None):
    prof = O.default_profiles(vocab)["cheap"]
    O.set_threads(threads or os.cpu_count() or 1)
    n = h["oids"].size
    dup = O.dup_flags(h["fids"], h["sigs"], 0.01)
    keep = ~dup
    topk = np.zeros((n, k), np.int32)
    topk[keep] = O.classify_topk(prof, seed, h["oids"][keep], h["true_class"][keep], k)
    return O.ingest(h["oids"], h["fids"], h["sigs"], h["feats"], topk, k, t, m, is_dup=dup)


def derive_k(ref, k: int):
    """The oracle result of the same stream ingested with a smaller K.

    Clustering never reads the top-K (tuner.py:10-12), top(K) is a prefix of
    the ranked list (core.py:60-61) and a class's best rank is the minimum
    position over the members' lists (clustering.py:65-69), so the K-run's
    top-K rows are the first K columns and its class sets are the entries of
    rank <= K.  One oracle run at the largest K checks every smaller K."""
    from dataclasses import replace
    cl = [replace(c, class_best_rank={cc: r for cc, r in c.class_best_rank.items() if r <= k})
          for c in ref.clusters]
    return replace(ref, topk=np.ascontiguousarray(ref.topk[:, :k]), clusters=cl)


def compare(dev: dict, ref, vocab: int) -> dict:
    """Field-by-field mismatch counts (0 everywhere = bit-exact)."""
    mism = {}
    n = ref.cluster_of.size
    keep = ~ref.is_dup
    mism["is_dup"] = int(np.count_nonzero(dev["is_dup"] != ref.is_dup))
    tk_ref = np.where(ref.topk == O.OTHER_CLASS, vocab, ref.topk)
    mism["topk_rows"] = int(np.count_nonzero((dev["topk"][keep] != tk_ref[keep]).any(axis=1)))
    mism["cluster_of"] = int(np.count_nonzero(dev["cluster_of"] != ref.cluster_of))
    mism["distance_computations"] = int(dev["dc"] != ref.distance_computations)
    C = len(ref.clusters)
    mism["n_clusters"] = int(dev["cluster_ids"].size != C)
    cen_bad = rep_bad = mem_bad = cls_bad = 0
    if dev["cluster_ids"].size == C:
        mism["cluster_ids"] = int(np.count_nonzero(dev["cluster_ids"] != np.arange(C)))
        cen = dev["centroids"].view(np.uint64)
        mo, co = dev["mem_off"], dev["cls_off"]
        for i, c in enumerate(ref.clusters):
            if not np.array_equal(cen[i], np.asarray(c.centroid, np.float64).view(np.uint64)):
                cen_bad += 1
            r = -1 if c.centroid_member_id is None else c.centroid_member_id
            rep_bad += int(dev["reps"][i] != r)
            a, b = mo[i], mo[i + 1]
            if (not np.array_equal(dev["mem_oid"][a:b], np.asarray(c.member_object_ids, np.int64))
                    or not np.array_equal(dev["mem_fid"][a:b], np.asarray(c.frame_ids, np.int64))):
                mem_bad += 1
            ca, cb = co[i], co[i + 1]
            got = dict(zip(dev["cls_id"][ca:cb].tolist(), dev["cls_rank"][ca:cb].tolist()))
            want = {(vocab if cc == O.OTHER_CLASS else cc): rr for cc, rr in c.class_best_rank.items()}
            cls_bad += int(got != want)
    mism.update(centroid_bits=cen_bad, representatives=rep_bad, members=mem_bad, class_ranks=cls_bad)
    post = O.build_postings(ref.clusters)
    po, pc = dev["post_off"], dev["post_cluster"]
    bad = 0
    for cls in range(vocab + 1):
        want = post.get(O.OTHER_CLASS if cls == vocab else cls, [])
        if pc[po[cls]:po[cls + 1]].tolist() != want:
            bad += 1
    mism["postings_classes"] = bad
    total = int(sum(mism.values()))
    return dict(objects_checked=int(n), classified=int(keep.sum()), clusters=C, mismatches=total,
                mismatch_by_field={k: v for k, v in mism.items() if v},
                distance_computations=int(ref.distance_computations),
                margin_objects={"within_1e-5_of_T": ref.margin_t, "within_1e-5_of_tie": ref.margin_tie},
                device_exact_rechecks=dev.get("exact_rechecks"))


def check_synth(data, n: int, k: int, t: float, m: int, vocab: int, device: int = 0, threads=None,
                batch: int = 0) -> dict:
    """Device ingest vs oracle on the first n objects of `data`; returns the report."""
    import paper_1801_03493_b200 as fx
    t0 = time.perf_counter()
    dev = device_ingest(data, n, k, t, m, vocab, fx.make_default_profiles(vocab)["cheap"], device=device,
                        batch=batch)
    t1 = time.perf_counter()
    h = host_stream(data, n)
    ref = oracle_ingest(h, k, t, m, vocab, threads=threads)
    t2 = time.perf_counter()
    rep = compare(dev, ref, vocab)
    rep.update(config=dict(n=n, dim=data.dim, vocab=vocab, k=k, t=t, m=m),
               device_s=round(t1 - t0, 3), oracle_s=round(t2 - t1, 3),
               oracle_threads=threads or os.cpu_count())
    return rep
