"""The native FOCUSIDX/1 reader (csrc/index_read.cu) against the reference's
own index.load (index.py:131-204): golden files written by the reference,
and mutated files (valid CRC re-stamped) that walk every error branch in the
reference's evaluation order.  CPU only (the reader is host code); the
reference comparison runs where /root/reference is importable."""

import os
import sys
import zlib

import numpy as np
import pytest

import paper_1801_03493_b200 as fx

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF_SRC = "/root/reference/pkg/src"


def _ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present")
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    from focusidx import index as ref_index
    return ref_index


def _stamp(body: str) -> str:
    return body + f"CRC32:{zlib.crc32(body.encode('utf-8')) & 0xFFFFFFFF:08x}\n"


def _body(path):
    text = open(path, encoding="utf-8").read()
    head, _, _ = text.rstrip("\n").rpartition("\n")
    return head + "\n"


def _same(a, b):
    from dataclasses import astuple
    assert astuple(a.header) == astuple(b.header)
    assert sorted(a.clusters) == sorted(b.clusters)
    assert list(a.clusters) == list(b.clusters)  # file order
    for cid, c in b.clusters.items():
        d = a.clusters[cid]
        assert np.asarray(d.centroid).view(np.uint64).tolist() == np.asarray(c.centroid).view(np.uint64).tolist()
        assert d.member_object_ids == c.member_object_ids and d.frame_ids == c.frame_ids
        assert d.class_best_rank == c.class_best_rank and list(d.class_best_rank) == list(c.class_best_rank)
        assert d.centroid_member_id == c.centroid_member_id
    assert a.postings == b.postings and list(a.postings) == list(b.postings)


@pytest.mark.parametrize("name", sorted(n for n in os.listdir(GOLD) if n.endswith(".focusidx")))
def test_golden_files_equal_reference_load(name):
    ref = _ref()
    path = os.path.join(GOLD, name)
    _same(fx.load(path), ref.load(path))


def _outcome(fn, path):
    try:
        return ("ok", fn(path))
    except Exception as e:  # noqa: BLE001 - the type is what is compared
        return ("err", type(e).__name__)


MUTATIONS = {
    "no_trailer": lambda b: b,
    "bad_crc": lambda b: b + "CRC32:00000000\n",
    "magic": lambda b: _stamp(b.replace("FOCUSIDX/1", "FOCUSIDX/2", 1)),
    "no_clusters": lambda b: _stamp(b.replace("[CLUSTERS]\n", "", 1).split("[POSTINGS]")[0]),
    "bad_header_int": lambda b: _stamp(b.replace("\nD=", "\nD=x", 1)),
    "header_missing_key": lambda b: _stamp("\n".join(l for l in b.split("\n") if not l.startswith("n=")) ),
    "header_underscore_ws": lambda b: _stamp(b.replace("\nD=", "\nD= 0_0", 1)),
    "record_parts": lambda b: _stamp(b.replace("[CLUSTERS]\n", "[CLUSTERS]\n1|2|3\n", 1)),
    "record_bad_cid": lambda b: _stamp(b.replace("[CLUSTERS]\n", "[CLUSTERS]\nx|||||\n", 1)),
    "dup_cid": lambda b: _stamp(b.replace("[POSTINGS]", b.split("[CLUSTERS]\n")[1].split("\n")[0] + "\n[POSTINGS]",
                                          1)),
    "no_postings": lambda b: _stamp(b.split("[POSTINGS]")[0]),
    "crlf": lambda b: _stamp(b).replace("\n", "\r\n"),
    "posting_bad_class": lambda b: _stamp(b + "99999|1\n"),
    "posting_bad_id": lambda b: _stamp(b + "0|a\n"),
    "posting_repeat": lambda b: _stamp(b + b.split("[POSTINGS]\n")[1].split("\n")[0] + "\n"),
}


@pytest.mark.parametrize("mut", sorted(MUTATIONS))
@pytest.mark.parametrize("name", ["index_small_d64.focusidx", "index_edge.focusidx"])
def test_mutated_files_match_reference(tmp_path, name, mut):
    ref = _ref()
    text = MUTATIONS[mut](_body(os.path.join(GOLD, name)))
    p = tmp_path / "m.focusidx"
    p.write_bytes(text.encode("utf-8"))
    got, want = _outcome(fx.load, str(p)), _outcome(ref.load, str(p))
    assert got[0] == want[0], (got, want)
    if got[0] == "ok":
        _same(got[1], want[1])
    else:
        assert got[1] == want[1]


def test_record_field_errors_in_reference_order(tmp_path):
    ref = _ref()
    base = _body(os.path.join(GOLD, "index_small_d64.focusidx"))
    first = base.split("[CLUSTERS]\n")[1].split("\n")[0]
    parts = first.split("|")
    variants = {
        "rank_not_int": parts[:5] + ["3:x"],
        "class_out_of_vocab": parts[:5] + ["100000:1"],
        "rank_bad_and_class_bad": parts[:5] + ["100000:x"],
        "centroid_not_float": parts[:2] + ["1.0,abc"] + parts[3:],
        "centroid_hex": parts[:2] + ["0x1p3"] + parts[3:],
        "centroid_inf_nan_ws": parts[:2] + [" inf,-Infinity, nan ,1_0.5"] + parts[3:],
        "members_empty": parts[:3] + [""] + parts[4:],
        "cmid_bad": parts[:1] + ["7a"] + parts[2:],
        "cmid_empty": parts[:1] + [""] + parts[2:],
        "ranks_repeat": parts[:5] + ["3:2,3:1,5:4"],
    }
    for tag, fields in variants.items():
        text = _stamp(base.replace(first, "|".join(fields), 1))
        p = tmp_path / f"{tag}.focusidx"
        p.write_bytes(text.encode("utf-8"))
        got, want = _outcome(fx.load, str(p)), _outcome(ref.load, str(p))
        assert got[0] == want[0], (tag, got, want)
        if got[0] == "ok":
            _same(got[1], want[1])
        else:
            assert got[1] == want[1], (tag, got, want)
