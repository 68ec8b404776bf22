"""Exception taxonomy of the drop-in API.

Same class names and hierarchy as the reference (focusidx/errors.py:4-95) so
callers' ``except`` clauses keep working; each C-ABI status code maps onto
one class (include/focus_b200.h).
"""


class FocusError(Exception):
    """Root of every error raised by this package."""


class UsageError(FocusError):
    """The caller passed bad arguments or parameters."""


class DataError(FocusError):
    """Input data or files are malformed or inconsistent."""


class UnknownProfile(UsageError):
    pass


class KOutOfRange(UsageError):
    pass


class NonPositiveM(UsageError):
    pass


class MissingTrueClass(DataError):
    pass


class EmptyHistogram(UsageError):
    pass


class DimensionMismatch(DataError):
    pass


class SignatureLengthMismatch(DataError):
    pass


class DuplicateClusterId(DataError):
    pass


class FormatVersionMismatch(DataError):
    pass


class ChecksumMismatch(DataError):
    pass


class KxTooLarge(UsageError):
    pass


class UnknownClass(UsageError):
    pass


class NonMonotoneSchedule(UsageError):
    pass


class DeviceError(FocusError):
    """CUDA failure, missing device, or the native library is not built."""


# fx_status -> exception class (include/focus_b200.h)
STATUS = {
    1: UsageError,
    2: DataError,
    3: ValueError,
    10: UnknownProfile,
    11: KOutOfRange,
    12: NonPositiveM,
    20: MissingTrueClass,
    30: DimensionMismatch,
    31: SignatureLengthMismatch,
    40: DuplicateClusterId,
    41: FormatVersionMismatch,
    42: ChecksumMismatch,
    50: KxTooLarge,
    51: UnknownClass,
    52: NonMonotoneSchedule,
    60: KeyError,
    90: DeviceError,
    91: DeviceError,
    99: DeviceError,
}
