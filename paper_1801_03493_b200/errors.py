"""Exception taxonomy of the drop-in API.

Same class names and hierarchy as the reference (focusidx/errors.py:4-95).
When the reference package is importable (the drop-in situation: a
``focusidx`` user switches the hot path to this package) the classes ARE the
reference's -- ``except focusidx.errors.KxTooLarge`` and
``pytest.raises(focusidx.errors.KxTooLarge)`` catch what this package raises.
Otherwise an identical local hierarchy is defined.  Each C-ABI status code
maps onto one class (include/focus_b200.h).
"""

try:  # the reference's own classes (types only; nothing else is imported)
    from focusidx import errors as _ref  # type: ignore
except Exception:  # pragma: no cover - depends on the environment
    _ref = None

# name -> base class name (focusidx/errors.py:4-95)
_TAXONOMY = (
    ("FocusError", None),
    ("UsageError", "FocusError"),
    ("DataError", "FocusError"),
    ("UnknownProfile", "UsageError"),
    ("KOutOfRange", "UsageError"),
    ("NonPositiveM", "UsageError"),
    ("MissingTrueClass", "DataError"),
    ("EmptyHistogram", "UsageError"),
    ("DimensionMismatch", "DataError"),
    ("SignatureLengthMismatch", "DataError"),
    ("DuplicateClusterId", "DataError"),
    ("FormatVersionMismatch", "DataError"),
    ("ChecksumMismatch", "DataError"),
    ("KxTooLarge", "UsageError"),
    ("UnknownClass", "UsageError"),
    ("NonMonotoneSchedule", "UsageError"),
    ("EmptySample", "UsageError"),
    ("NoViableConfig", "FocusError"),
    ("EmptyViableSet", "UsageError"),
    ("InvalidSpec", "UsageError"),
)

_ns = globals()
for _name, _base in _TAXONOMY:
    _cls = getattr(_ref, _name, None) if _ref is not None else None
    if _cls is None:
        _cls = type(_name, (Exception if _base is None else _ns[_base],),
                    {"__module__": __name__, "__doc__": f"focusidx.errors.{_name} (drop-in)"})
    _ns[_name] = _cls

SHARES_REFERENCE_CLASSES = _ref is not None


class DeviceError(FocusError):  # noqa: F821 - defined by the loop above
    """CUDA failure, missing device, or the native library is not built."""


# fx_status -> exception class (include/focus_b200.h)
STATUS = {
    1: UsageError,  # noqa: F821
    2: DataError,  # noqa: F821
    3: ValueError,
    10: UnknownProfile,  # noqa: F821
    11: KOutOfRange,  # noqa: F821
    12: NonPositiveM,  # noqa: F821
    20: MissingTrueClass,  # noqa: F821
    30: DimensionMismatch,  # noqa: F821
    31: SignatureLengthMismatch,  # noqa: F821
    40: DuplicateClusterId,  # noqa: F821
    41: FormatVersionMismatch,  # noqa: F821
    42: ChecksumMismatch,  # noqa: F821
    50: KxTooLarge,  # noqa: F821
    51: UnknownClass,  # noqa: F821
    52: NonMonotoneSchedule,  # noqa: F821
    60: KeyError,
    90: DeviceError,
    91: DeviceError,
    99: DeviceError,
}

__all__ = [n for n, _ in _TAXONOMY] + ["DeviceError", "STATUS", "SHARES_REFERENCE_CLASSES"]
