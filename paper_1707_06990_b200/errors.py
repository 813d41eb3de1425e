"""Exception hierarchy mirroring denseplan/errors.hpp:8-61.

C-ABI status codes 1..12 map to these classes in declaration order; codes
>= 100 are device (CUDA/NCCL) failures.
"""


class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class BoundsError(Error):
    pass


class SizeOverflowError(Error):
    pass


class CapacityError(Error):
    pass


class AccountingError(Error):
    pass


class ConfigError(Error):
    pass


class FormatError(Error):
    pass


class LabelError(Error):
    pass


class DegenerateBatchError(Error):
    pass


class ProtocolError(Error):
    pass


class RangeError(Error):
    pass


class VerifyError(Error):
    pass


class DeviceError(Error):
    """CUDA (100) or NCCL (101) failure reported through the C ABI."""


_BY_STATUS = {1: ShapeError, 2: BoundsError, 3: SizeOverflowError, 4: CapacityError,
              5: AccountingError, 6: ConfigError, 7: FormatError, 8: LabelError,
              9: DegenerateBatchError, 10: ProtocolError, 11: RangeError, 12: VerifyError}


def from_status(code: int, msg: str) -> Error:
    cls = _BY_STATUS.get(code, DeviceError if code >= 100 else Error)
    return cls(f"[status {code}] {msg}")
