"""Error taxonomy of the reference, raised from C-ABI status codes.

Names and base classes follow rowfuse/core.py:25-46 so code written against
the reference catches the same exceptions here.
"""


class SizeMismatch(ValueError):
    """Buffer length or dimension does not match the declared shape (rowfuse/core.py:25-26)."""


class ShapeMismatch(ValueError):
    """Two operands disagree on shape or dtype (rowfuse/core.py:29-30)."""


class NonContiguousInput(ValueError):
    """A kernel received a non-contiguous view (rowfuse/core.py:33-38)."""


class OddHeadDim(ValueError):
    """Rotary embedding requires an even head dimension (rowfuse/core.py:41-42)."""


class TargetOutOfRange(IndexError):
    """A class index falls outside [0, vocab) (rowfuse/core.py:45-46)."""


class UnsupportedOption(NotImplementedError):
    """A Liger option this build does not implement yet."""


class CudaError(RuntimeError):
    """Kernel launch or CUDA runtime failure inside the library."""


class ExtensionMissing(RuntimeError):
    """The sm_100a library is not built or cannot be loaded. There is no fallback."""


STATUS = {
    1: NonContiguousInput,
    2: ShapeMismatch,
    3: SizeMismatch,
    4: OddHeadDim,
    5: TargetOutOfRange,
    6: UnsupportedOption,
    7: CudaError,
    8: ValueError,
}
