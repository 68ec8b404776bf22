"""Shared boundary types for the drop-in.

When the reference package is importable (a focusidx user switching the hot
path to this package), the plain data records that cross the API -- objects,
configs, profiles, headers, clusters, reports, query requests/results --
ARE the reference's classes, so values built on either side compare equal
and isinstance checks keep working (the error classes follow the same rule,
errors.py).  Only type definitions are taken from focusidx; no reference
code runs on the hot path.  Without focusidx the package's own identical
records are used.
"""

from __future__ import annotations

import importlib


def shared(module: str, name: str, own):
    """focusidx.<module>.<name> when importable, else `own`."""
    try:
        mod = importlib.import_module(f"focusidx.{module}")
    except Exception:
        return own
    return getattr(mod, name, own)
