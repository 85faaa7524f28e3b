"""Input coercion at the reference-facing boundary.

The reference coerces every input to a C-contiguous float64 numpy array and raises
``ShapeError`` (a ``ValueError``) on a wrong rank (numerics.py:17-26).  This module does
the B200 equivalent: inputs become CUDA tensors viewed as [B, H, N, d] (rank 2 = the
reference's single-head [N, d]; rank 4 = the batched extension), and results go back in
the caller's container (numpy in -> numpy float64 out, torch in -> torch out).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


class ShapeError(ValueError):
    """Operand dimensions are incompatible (numerics.py:17-18)."""


def num_blocks(n: int, block: int) -> int:
    """ceil(n / block) (numerics.py:68-69)."""
    return -(-n // block)


@dataclass(frozen=True)
class Boundary:
    """How the caller handed us a tensor, so results can be returned the same way."""

    rank: int
    numpy: bool
    device: torch.device


def current_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_13515_b200 requires a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def to_device4(x, dtype: torch.dtype | None, name: str, device: torch.device | None = None):
    """Return (tensor [B,H,N,d] on CUDA, Boundary).  ``dtype=None`` keeps a floating dtype."""
    is_np = not isinstance(x, torch.Tensor)
    t = torch.as_tensor(np.asarray(x)) if is_np else x
    if t.dim() not in (2, 4):
        raise ShapeError(f"{name}: expected rank 2 [N,d] or rank 4 [B,H,N,d], got rank {t.dim()} "
                         f"with shape {tuple(t.shape)}")
    if t.shape[-1] < 1 or t.shape[-2] < 1:
        raise ShapeError(f"{name}: empty tensor {tuple(t.shape)}")
    if device is None:
        device = t.device if t.is_cuda else current_device()
    _lib.require_device(device)
    want = dtype if dtype is not None else (t.dtype if t.dtype in _lib.DTYPE_CODES else torch.float64)
    t = t.to(device=device, dtype=want, non_blocking=True)
    if t.stride(-1) != 1:
        t = t.contiguous()
    rank = t.dim()
    if rank == 2:
        t = t.view(1, 1, *t.shape) if t.is_contiguous() else t.contiguous().view(1, 1, *t.shape)
    return t, Boundary(rank=rank, numpy=is_np, device=device)


def from_device(t: torch.Tensor, b: Boundary, rows_dims: int = 2):
    """Undo ``to_device4``'s batching for an output whose trailing ``rows_dims`` axes are
    per-head (e.g. 2 for [N,d], 1 for lse [N])."""
    if b.rank == 2:
        t = t.reshape(t.shape[-rows_dims:])
    if b.numpy:
        return t.detach().to(torch.float64).cpu().numpy()
    return t


class FiniteGuard:
    """Deferred finiteness verdicts (the reference's ``ensure_finite``, numerics.py:29-32).

    The scans run on the GPU (K0 ``spa2_check_finite`` for v / dO, K1's pooling for q / k)
    and store 1 into a flag that lives in pinned, device-mapped HOST memory (the kernels write
    it over PCIe only when they find a NaN/Inf), so no copy is enqueued — a D2H copy on the
    compute stream would queue behind bulk transfers on the copy engine.  An event recorded
    after the scans says when the flag is final.  The verdict is enforced

    * immediately (``block=True``) for numpy callers, whose results are synchronised
      anyway, and for ``check_finite="sync"``;
    * otherwise without a host sync: the backward pass of the same call and every later
      operator call enforce the verdicts that have landed by then, ``check_pending()``
      forces all outstanding ones.

    A non-finite input thus raises ``FloatingPointError`` as in the reference, for torch
    callers possibly one call later (the output of the offending call is then non-finite).
    """

    def __init__(self):
        self._pending: list[tuple[torch.cuda.Event, torch.Tensor, str]] = []

    @staticmethod
    def new_flag(device: torch.device) -> torch.Tensor:
        """A zeroed int32 flag in pinned host memory (UVA: the same pointer is valid in
        kernels).  It stays referenced until its verdict is enforced, so the pinned block is
        not recycled while a kernel may still write it."""
        return torch.zeros((1,), dtype=torch.int32, pin_memory=True)

    def submit(self, flag: torch.Tensor, what: str, block: bool, device: torch.device | None = None,
               extra_event: torch.cuda.Event | None = None) -> tuple:
        """Register ``flag`` (written by kernels on the current stream, and by those before
        ``extra_event`` on a side stream) as the verdict on ``what``."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(device))
        entry = (_Events(ev, extra_event), flag, what)
        if block:
            self._verify(entry)
        else:
            self._pending.append(entry)
        return entry

    @staticmethod
    def _verify(entry) -> None:
        ev, host, what = entry
        ev.synchronize()
        if int(host[0]) != 0:
            raise FloatingPointError(f"non-finite values in {what}")

    def resolve(self, entry, block: bool = False) -> None:
        """Enforce one verdict if it has landed (or wait for it with ``block``); used by the
        backward pass of the call that made it."""
        if entry in self._pending and (block or entry[0].query()):
            self._pending.remove(entry)
            self._verify(entry)

    def check_pending(self, block: bool = True) -> None:
        """Enforce outstanding verdicts: all of them (block=True) or the completed ones."""
        keep = []
        err = None
        for entry in self._pending:
            if block or entry[0].query():
                try:
                    self._verify(entry)
                except FloatingPointError as e:
                    err = err or e
            else:
                keep.append(entry)
        self._pending = keep
        if err is not None:
            raise err


class _Events:
    """Both events of a verdict (current stream, optional side stream) behave as one."""

    def __init__(self, a: torch.cuda.Event, b: torch.cuda.Event | None):
        self.a, self.b = a, b

    def query(self) -> bool:
        return self.a.query() and (self.b is None or self.b.query())

    def synchronize(self) -> None:
        self.a.synchronize()
        if self.b is not None:
            self.b.synchronize()


finite_guard = FiniteGuard()


def check_pending() -> None:
    """Raise ``FloatingPointError`` now if any earlier call's inputs were non-finite."""
    finite_guard.check_pending(block=True)


def make_rng(seed: int) -> np.random.Generator:
    """PCG64 generator, bit-identical streams on every platform (numerics.py:78-79)."""
    return np.random.Generator(np.random.PCG64(seed))


def format_float(v: float) -> str:
    """Shortest round-trip decimal form (numerics.py:122-124)."""
    return repr(float(v))
