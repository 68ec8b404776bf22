"""FOCUSIDX/1 index files (index.py:88-204): the native
writer (fx_index_write, host-only) must reproduce the bytes the reference's
index.save wrote (tests/golden/index_*.focusidx, tools/gen_golden_index.py),
and load must raise the reference's errors.  CPU only."""

import json
import os
import zlib

import numpy as np
import pytest

fx = pytest.importorskip("paper_1801_03493_b200")
from paper_1801_03493_b200 import index as fxi  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(f for f in os.listdir(GOLDEN) if f.startswith("index_") and f.endswith(".focusidx"))


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name", FILES)
def test_load_save_round_trip_is_byte_identical(name, tmp_path):
    src = os.path.join(GOLDEN, name)
    idx = fxi.load(src)
    out = tmp_path / "re.focusidx"
    fxi.save(idx, str(out), threads=3)
    assert _bytes(out) == _bytes(src)


def test_writer_renders_fresh_clusters_like_the_reference(tmp_path):
    with open(os.path.join(GOLDEN, "index_edge.json")) as fh:
        d = json.load(fh)
    h = d["header"]
    cfg = fx.Config(h["config"]["profile_id"], k=h["config"]["k"], l_s=h["config"]["l_s"], t=h["config"]["t"],
                    m=h["config"]["m"])
    header = fx.IndexHeader(h["stream_id"], h["dim"], h["vocab"], h["n_objects"], cfg)
    clusters = {}
    for c in d["clusters"]:
        clusters[c["cluster_id"]] = fx.Cluster(
            cluster_id=c["cluster_id"], centroid=np.array([float.fromhex(x) for x in c["centroid"]]),
            member_object_ids=c["members"], frame_ids=c["frames"], class_best_rank={k: v for k, v in c["ranks"]},
            centroid_member_id=c["rep"], sealed=True)
    postings = {k: v for k, v in d["postings"]}
    idx = fx.TopKIndex(header, clusters=clusters, postings=postings)
    out = tmp_path / "edge.focusidx"
    fx.save(idx, str(out))
    assert _bytes(out) == _bytes(os.path.join(GOLDEN, "index_edge.focusidx"))


def _with_crc(body: str) -> str:
    return body + f"CRC32:{zlib.crc32(body.encode('utf-8')) & 0xFFFFFFFF:08x}\n"


def test_load_errors_match_reference(tmp_path):
    text = _bytes(os.path.join(GOLDEN, "index_gt_d8.focusidx")).decode()
    body = text[:text.rindex("CRC32:")]
    p = tmp_path / "x.focusidx"
    p.write_text(body + "CRC32:00000000\n")
    with pytest.raises(fx.ChecksumMismatch):
        fxi.load(str(p))
    p.write_text(body)
    with pytest.raises(fx.ChecksumMismatch):
        fxi.load(str(p))
    p.write_text(_with_crc(body.replace("FOCUSIDX/1", "FOCUSIDX/2", 1)))
    with pytest.raises(fx.FormatVersionMismatch):
        fxi.load(str(p))
    lines = body.splitlines(keepends=True)
    first = next(i for i, ln in enumerate(lines) if ln.startswith("[CLUSTERS]")) + 1
    p.write_text(_with_crc("".join(lines[:first + 1] + [lines[first]] + lines[first + 1:])))
    with pytest.raises(fx.DuplicateClusterId):
        fxi.load(str(p))
    p.write_text(_with_crc("".join(ln for ln in lines if not ln.startswith("[POSTINGS]"))))
    with pytest.raises(fx.DataError):
        fxi.load(str(p))


def test_config_text_round_trip():
    cfg = fx.Config("cheap+spec6", k=3, l_s=6, t=0.8, m=25)
    text = fx.format_config(cfg)
    assert text.splitlines()[3] == "t=0.800000"
    back = fx.parse_config("# comment\n\n" + text)
    assert (back.profile_id, back.k, back.l_s, back.t, back.m) == ("cheap+spec6", 3, 6, 0.8, 25)
    with pytest.raises(fx.DataError):
        fx.parse_config("profile=cheap\nk=3\n")
