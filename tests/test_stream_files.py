"""FOCUSSTREAM/1 stream files (streamio.py): the native
decoder (fx_stream_file_*, host threads) against the reference semantics --
Python float()/int() per field -- on a file the reference's write_stream
produced (tests/golden/stream_gt_d8.focusstream, tools/gen_golden_stream.py),
and the reference's errors for malformed files.  CPU only."""

import os

import numpy as np
import pytest

fx = pytest.importorskip("paper_1801_03493_b200")
from paper_1801_03493_b200 import streamio  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "stream_gt_d8.focusstream")


def _py_parse(path):
    """The reference read_stream's field parsing (streamio.py:58-113)."""
    lines = open(path, encoding="utf-8").read().splitlines()
    body = lines.index("[OBJECTS]") + 1
    kv = dict(ln.partition("=")[::2] for ln in lines[1:body - 1])
    V = int(kv["V"])
    rows = []
    for ln in lines[body:]:
        if not ln:
            continue
        p = ln.split("|")
        tc = -2 if p[2] == "" else (-1 if int(p[2]) == V else int(p[2]))
        rows.append((int(p[0]), int(p[1]), tc, [float(x) for x in p[3].split(",")],
                     [float(x) for x in p[4].split(",")]))
    return kv, rows


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_decode_matches_python_float_parsing(threads):
    kv, rows = _py_parse(GOLDEN)
    header, a = streamio.read_stream_arrays(GOLDEN, threads=threads)
    assert (header.stream_id, header.fps, header.dim, header.sig_dim, header.vocab) == \
        (kv["stream_id"], float(kv["fps"]), int(kv["D"]), int(kv["S"]), int(kv["V"]))
    assert a["object_ids"].tolist() == [r[0] for r in rows]
    assert a["frame_ids"].tolist() == [r[1] for r in rows]
    assert a["true_class"].tolist() == [r[2] for r in rows]
    assert -2 in a["true_class"] and -1 in a["true_class"]
    sig = np.array([r[3] for r in rows])
    feat = np.array([r[4] for r in rows])
    assert np.array_equal(a["pixel_signatures"].view(np.uint64), sig.view(np.uint64))
    assert np.array_equal(a["features"].view(np.uint64), feat.view(np.uint64))
    _, a32 = streamio.read_stream_arrays(GOLDEN, feat_dtype=np.float32)
    assert np.array_equal(a32["features"], feat.astype(np.float32))


def test_read_stream_objects_and_rewrite_round_trip(tmp_path):
    header, objs = streamio.read_stream(GOLDEN)
    assert objs[5].true_class is None and objs[11].true_class == fx.OTHER_CLASS
    assert objs[3].timestamp_s == objs[3].frame_id / header.fps
    out = tmp_path / "re.focusstream"
    streamio.write_stream(str(out), header, objs)
    assert out.read_bytes() == open(GOLDEN, "rb").read()


def _body(path):
    text = open(path, encoding="utf-8").read()
    head, _, body = text.partition("[OBJECTS]\n")
    return head, body.splitlines()


@pytest.mark.parametrize("mutate,exc", [
    (lambda h, b: ("FOCUSSTREAM/2" + h[13:], b), fx.FormatVersionMismatch),
    (lambda h, b: (h.replace("D=8\n", ""), b), fx.DataError),
    (lambda h, b: (h, b[:3] + ["1|2|3"] + b[3:]), fx.DataError),
    (lambda h, b: (h, b[:3] + [b[3].replace(",", ",x", 1)] + b[4:]), ValueError),
    (lambda h, b: (h, b[:3] + [b[3].rsplit(",", 1)[0]] + b[4:]), fx.DataError),
    (lambda h, b: (h, b[:3] + [b[3].replace(b[3].split("|")[2], "77", 1) if b[3].split("|")[2] else b[3]] + b[4:]),
     fx.DataError),
    (lambda h, b: (h, b[:4] + [b[2]] + b[4:]), fx.DataError),
])
def test_malformed_files_raise_reference_errors(tmp_path, mutate, exc):
    h, b = _body(GOLDEN)
    h2, b2 = mutate(h, b)
    p = tmp_path / "bad.focusstream"
    p.write_text(h2 + ("[OBJECTS]\n" if "[OBJECTS]" not in h2 else "") + "\n".join(b2) + "\n")
    with pytest.raises(exc):
        streamio.read_stream_arrays(str(p))
