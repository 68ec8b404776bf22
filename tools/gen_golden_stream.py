"""Golden FOCUSSTREAM/1 file written by the UNMODIFIED
reference `focusidx.streamio.write_stream`, for tests/test_stream_files.py.
Run in the build container:  python tools/gen_golden_stream.py

The gt_d8 golden stream (tools/gen_golden.py CASES), with a few objects made
unlabeled and one labeled OTHER so both encodings of true_class appear."""
import dataclasses
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "tools"))

from focusidx import simharness, streamio  # noqa: E402
from focusidx.core import OTHER_CLASS  # noqa: E402

from gen_golden import CASES  # noqa: E402

spec_kw = next(c[1] for c in CASES if c[0] == "gt_d8")
header, objects = simharness.generate_stream(simharness.StreamSpec(**spec_kw))
objs = []
for i, o in enumerate(objects):
    if i % 97 == 5:
        o = dataclasses.replace(o, true_class=None)
    elif i == 11:
        o = dataclasses.replace(o, true_class=OTHER_CLASS)
    objs.append(o)
path = os.path.join(REPO, "tests", "golden", "stream_gt_d8.focusstream")
streamio.write_stream(path, header, objs)
print(path, os.path.getsize(path), "bytes")
