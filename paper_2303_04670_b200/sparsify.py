"""Error-feedback sparsification (mirrors evincr/sparsify.py).

Rounds the residual-corrected increment to multiples of k on the GPU and
carries the round-off forward (sparsify.py:54-78).  The per-op
``sparsify_step`` exposes ``norm_ema``/``k`` as Python floats like the
reference, but keeps them as a device float64 pair that is read back only when
an attribute is read (the operators never synchronise the host); the Graph
runtime keeps them as device float64 scalars.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .tensors import IncrementTensor, TileMask, TileShape, as_tensor, grid_shape, make_tile_mask

__all__ = ["SparsifyState", "sparsify_step"]


class SparsifyState:
    """Residual tensor, rolling input norm and rounding step (sparsify.py:22-51)."""

    def __init__(self, shape, tp: float = 0.0, ema_decay: float = 0.9, k: float = 0.0):
        if tp < 0:
            raise ValueError("threshold parameter must be >= 0")
        if not (0.0 < ema_decay < 1.0):
            raise ValueError("ema_decay must lie in (0, 1)")
        self.shape = tuple(int(v) for v in shape)
        self.tp = float(tp)
        self.ema_decay = float(ema_decay)
        self.delta = torch.zeros(self.shape, dtype=torch.float32, device="cuda")
        self._sc = torch.tensor([0.0, float(k)], dtype=torch.float64, device="cuda")  # (norm_ema, k)

    @property
    def norm_ema(self) -> float:
        return float(self._sc[0].item())

    @norm_ema.setter
    def norm_ema(self, v: float) -> None:
        self._sc[0] = float(v)

    @property
    def k(self) -> float:
        return float(self._sc[1].item())

    @k.setter
    def k(self, v: float) -> None:
        self._sc[1] = float(v)

    def _fold(self, sc) -> None:
        """Take norm_ema (and k when t_p > 0, sparsify.py:76) from a device pair the kernel updated."""
        if self.tp > 0:
            self._sc.copy_(sc)
        else:
            self._sc[0:1].copy_(sc[0:1])

    def reset(self, dense_input) -> None:
        """Clear the residual and seed the norm at a dense pass (sparsify.py:43-51)."""
        x = as_tensor(dense_input)
        if tuple(x.shape) != self.shape:
            raise ValueError(f"dense input {tuple(x.shape)} vs state {self.shape}")
        self.delta = torch.zeros(self.shape, dtype=torch.float32, device=x.device)
        nb = 64
        part = torch.empty(nb, dtype=torch.float64, device=x.device)
        sc = self._sc.clone()
        lib = _lib.lib()
        s = _lib.stream_ptr()
        _lib.check(lib.evc_sumsq_dense(_lib.ptr(x), 0, x.numel(), _lib.ptr(part), nb, 1, s), "sumsq")
        _lib.check(lib.evc_sparsify_finalize(_lib.ptr(part), nb, _lib.ptr(sc), _lib.ptr(sc) + 8, self.tp,
                                             self.ema_decay, 1, 1, s), "sparsify_finalize")
        self._fold(sc)


def sparsify_step(x: IncrementTensor, state: SparsifyState) -> IncrementTensor:
    """Round the corrected increment to multiples of k; keep the residual (sparsify.py:54-78)."""
    if x.shape != state.shape:
        raise ValueError(f"increment {x.shape} vs state {state.shape}")
    dev = x.values.device
    tile: TileShape = x.tile
    c, h, w = x.shape
    dlive = make_tile_mask(state.delta, tile).u8.clone()
    yv = torch.zeros(x.shape, dtype=torch.float32, device=dev)
    yf = torch.zeros(grid_shape(x.shape, tile), dtype=torch.uint8, device=dev)
    lib = _lib.lib()
    dx = x.desc()
    part = torch.zeros(int(lib.evc_sparsify_partials(dx)), dtype=torch.float64, device=dev)
    sc = state._sc.clone()
    s = _lib.stream_ptr()
    dy = _lib.tdesc(_lib.ptr(yv), _lib.ptr(yf), 0, 0, c, h, w, tile.h, tile.w)
    ticket = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.evc_sparsify(dx, _lib.ptr(state.delta), 0, _lib.ptr(dlive), dy, _lib.ptr(sc) + 8, _lib.ptr(sc),
                                state.tp, state.ema_decay, _lib.ptr(part), _lib.ptr(ticket), None, 0, 0, 0, None, 1, 0, 1, s),
               "sparsify")
    state._fold(sc)
    return IncrementTensor(yv, TileMask(yf, tile))
