"""Exception types mirroring /root/reference/proj/core/include/chunkode/errors.hpp:9-69.

The C ABI carries them as a cko_status plus a cko_error payload; raise_for()
turns that back into the matching exception, with the same location fields.
"""
from __future__ import annotations

from . import abi


class Error(RuntimeError):
    """chunkode::Error (errors.hpp:9-11)."""


class ShapeMismatch(Error):
    """errors.hpp:14-16."""


class SingularBlock(Error):
    """errors.hpp:20-28: chunk_index is the row within the chunk."""

    def __init__(self, chunk_index: int, batch_index: int, msg: str | None = None):
        super().__init__(msg or f"singular diagonal block at chunk row {chunk_index}, batch {batch_index}")
        self.chunk_index = chunk_index
        self.batch_index = batch_index


class SizeGuardExceeded(Error):
    """errors.hpp:31-34."""


class StrategyUnavailable(Error):
    """errors.hpp:36-39."""


class NonFiniteOutput(Error):
    """errors.hpp:41-44."""


class NewtonDivergence(Error):
    """errors.hpp:48-64."""

    def __init__(self, chunk_start_step, batch_index, iterations, residual_norm, initial_norm, msg=None):
        super().__init__(
            msg
            or f"Newton did not converge for chunk starting at step {chunk_start_step} (batch {batch_index}): "
            f"|r| = {residual_norm} after {iterations} iterations, |r0| = {initial_norm}"
        )
        self.chunk_start_step = chunk_start_step
        self.batch_index = batch_index
        self.iterations = iterations
        self.residual_norm = residual_norm
        self.initial_norm = initial_norm


class InvalidTimeGrid(Error):
    """errors.hpp:67-69."""


class DeviceError(Error):
    """CUDA / communication failure (no reference counterpart)."""


def raise_for(status: int, err: abi.CkoError) -> None:
    if status == abi.CKO_OK:
        return
    msg = err.msg.decode(errors="replace")
    if status == abi.CKO_SINGULAR_BLOCK:
        raise SingularBlock(err.chunk_index, err.batch_index, msg)
    if status == abi.CKO_NEWTON_DIVERGENCE:
        raise NewtonDivergence(err.chunk_start_step, err.batch_index, err.iterations,
                               err.residual_norm, err.initial_norm, msg)
    cls = {
        abi.CKO_SHAPE_MISMATCH: ShapeMismatch,
        abi.CKO_NON_FINITE: NonFiniteOutput,
        abi.CKO_STRATEGY_UNAVAILABLE: StrategyUnavailable,
        abi.CKO_SIZE_GUARD: SizeGuardExceeded,
        abi.CKO_INVALID_TIME_GRID: InvalidTimeGrid,
        abi.CKO_ERROR: Error,
    }.get(status, DeviceError)
    raise cls(msg)
