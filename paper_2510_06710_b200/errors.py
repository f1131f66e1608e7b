"""Exception taxonomy mirroring chunkrl/core/errors.hpp:9-48, keyed by ckrl status codes."""


class Error(RuntimeError):
    """chunkrl::Error — base of every engine error."""


class UnsupportedCombination(Error):
    pass


class GranularityOrderViolation(Error):
    pass


class LengthMismatch(Error):
    pass


class BadResetId(Error):
    pass


class HeadMismatch(Error):
    pass


class NonFinite(Error):
    pass


class DegenerateGroup(Error):
    pass


class SkipUpdate(Error):
    pass


class InvalidPlan(Error):
    pass


class MemoryOverflow(Error):
    pass


class EmptyTrace(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    """Device / launch failure (no reference counterpart: the reference has no device)."""


class InvalidArgument(Error):
    pass


class NcclError(Error):
    pass


_BY_STATUS = {
    1: UnsupportedCombination, 2: GranularityOrderViolation, 3: LengthMismatch, 4: BadResetId,
    5: HeadMismatch, 6: NonFinite, 7: DegenerateGroup, 8: SkipUpdate, 9: InvalidPlan,
    10: MemoryOverflow, 11: EmptyTrace, 12: ConfigError, 13: Error, 14: CudaError,
    15: InvalidArgument, 16: NcclError,
}


def from_status(status: int, msg: str = "") -> Error:
    cls = _BY_STATUS.get(int(status), Error)
    return cls(msg or cls.__name__)
