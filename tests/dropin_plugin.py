"""pytest plugin: the INTEGRATION.md §3 switch, as a maintainer would apply
it -- the reference package's hot-path entry points are replaced by this
package's before any test module imports them (the reference's tests bind
names at import time: ``from focusidx.ingest import ingest_stream``).

    python -m pytest -p dropin_plugin <reference tests>

Replaced: focusidx.ingest.{ingest_stream, pixel_diff},
focusidx.index.{build, lookup, save, load}, focusidx.query.QuerySession,
focusidx.tuner._GridEvaluator (the device grid evaluation).
Everything else (types, profiles, the rank-model classify, the tuner, the
simulator) stays the reference's.  This package's error classes are the
reference's own classes when focusidx is importable (errors.py), so the
tests' ``pytest.raises(focusidx.errors.X)`` catch what the drop-in raises.
"""

import focusidx  # noqa: F401  (first: errors.py aliases its classes)
from focusidx import index as _ref_index
from focusidx import ingest as _ref_ingest
from focusidx import query as _ref_query
from focusidx import tuner as _ref_tuner

import paper_1801_03493_b200 as fx

SWITCHED = []


def _switch(mod, name, new):
    setattr(mod, name, new)
    SWITCHED.append(f"{mod.__name__}.{name}")


_switch(_ref_ingest, "ingest_stream", fx.ingest_stream)
_switch(_ref_ingest, "pixel_diff", fx.pixel_diff)
_switch(_ref_index, "build", fx.build)
_switch(_ref_index, "lookup", fx.lookup)
_switch(_ref_index, "save", fx.save)
_switch(_ref_index, "load", fx.load)
_switch(_ref_query, "QuerySession", fx.QuerySession)
_switch(_ref_tuner, "_GridEvaluator", fx.tuner.GridEvaluator)
assert fx.errors.SHARES_REFERENCE_CLASSES, "the drop-in must raise the reference's error classes"


def pytest_report_header(config):
    return "focus drop-in switched: " + ", ".join(SWITCHED)
