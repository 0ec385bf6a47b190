"""Exception hierarchy of the reference (proj/include/rotavote/errors.hpp:8-55), mapped from
the C-ABI status codes (include/rotavote_b200.h rv_status)."""


class Error(RuntimeError):
    """rotavote::Error"""


class PoleProximity(Error):
    pass


class EmptyInput(Error):
    pass


class NoPeak(Error):
    pass


class DegenerateProjection(Error):
    pass


class NoVotes(Error):
    pass


class AllDegenerate(Error):
    pass


class RankDeficient(Error):
    pass


class NoConsensus(Error):
    pass


class InvalidConfig(Error):
    pass


class IoError(Error):
    pass


class EmptyFile(Error):
    pass


class ParseError(Error):
    """rotavote::ParseError: message "<what> (line N)", the 1-based line in .line."""

    def __init__(self, msg: str, line: int = 0):
        super().__init__(f"{msg} (line {line})")
        self.line = line


class DeviceError(Error):
    """CUDA / NCCL / allocation failures of the device path (no reference counterpart)."""


STATUS_TO_ERROR = {
    1: EmptyInput,
    2: NoPeak,
    3: DegenerateProjection,
    4: NoVotes,
    5: AllDegenerate,
    6: RankDeficient,
    7: NoConsensus,
    8: InvalidConfig,
    9: PoleProximity,
    10: DeviceError,
    11: DeviceError,
    15: ParseError,
    16: EmptyFile,
    17: IoError,
    12: DeviceError,
    13: DeviceError,
    14: DeviceError,
}

ERROR_NAMES = {code: cls.__name__ for code, cls in STATUS_TO_ERROR.items()}
