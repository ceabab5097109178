"""Oracle error classes (SPEC.md S:47 ConversionError, S:56 FormatError, S:65 LookupError)."""


class OracleError(Exception):
    pass


class InvalidError(OracleError):
    """Bad parameter (alignment / block size / chunk size) -- SURVEY §8(c) O1."""


class ConversionError(OracleError):
    """Duplicate/empty name, payload != prod(shape)*width, bad dtype/device."""


class FormatError(OracleError):
    """Malformed index (SURVEY §8(c) read-side validation)."""


class OracleLookupError(OracleError, KeyError):
    """Unknown tensor name."""


class ChecksumError(OracleError):
    """A recomputed block checksum differs from the index (O9(d))."""

    def __init__(self, partition: int, block: int):
        super().__init__(f"checksum mismatch in partition {partition}, block {block}")
        self.partition = partition
        self.block = block
