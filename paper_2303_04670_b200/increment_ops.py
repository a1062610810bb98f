"""Increment-domain operators (mirrors evincr/increment_ops.py).

Each operator maps an input increment to the output increment on the GPU
(libevconv.so).  Linear operators drop biases; nonlinear ones use an
accumulator of all increments since the last dense pass:
y = f(acc + dx) - f(acc).  Masks and FLOP meters follow the reference
bit-exactly; values match within float32 reassociation.

These per-op functions serve one session and allocate their outputs; the
Graph runtime drives the same kernels over preallocated, batched buffers.
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, tensors
from .tensors import (
    Activation,
    IncrementTensor,
    TileMask,
    TileShape,
    as_matrix,
    as_tensor,
    choose_splits,
    conv_geometry,
    conv_output_hw,
    grid_shape,
    make_tile_mask,
    pack_conv_weight,
)

__all__ = [
    "ConvParams",
    "AccState",
    "FlopCounter",
    "inc_conv2d",
    "inc_linear",
    "inc_add",
    "inc_activation",
    "inc_mul",
    "inc_concat",
    "inc_upsample",
    "inc_maxpool",
    "flatten_increment",
]


@dataclass(frozen=True)
class ConvParams:
    """Static convolution geometry (increment_ops.py:58-77)."""

    kernel: tuple
    c_in: int
    c_out: int
    stride: int = 1
    padding: int = 0

    def __post_init__(self):
        if self.stride < 1:
            raise ValueError("stride must be >= 1")
        if self.padding < 0:
            raise ValueError("padding must be >= 0")

    @classmethod
    def from_weight(cls, weight, stride: int = 1, padding: int = 0) -> "ConvParams":
        c_out, c_in, kh, kw = tuple(weight.shape)
        return cls((kh, kw), c_in, c_out, stride, padding)


class AccState:
    """Running sum of increments seen by a nonlinear node (increment_ops.py:80-94)."""

    __slots__ = ("x_acc",)

    def __init__(self, x_acc):
        self.x_acc = as_tensor(x_acc)

    @classmethod
    def zeros(cls, shape) -> "AccState":
        return cls(torch.zeros(shape, dtype=torch.float32, device="cuda"))

    def set_dense(self, x) -> None:
        self.x_acc = as_tensor(x).clone()

    def fold(self, dx) -> None:
        self.x_acc = self.x_acc + as_tensor(dx)


class FlopCounter:
    """2 ops per multiply-accumulate (increment_ops.py:97-113).

    Same fields and methods as the reference dataclass.  ``add`` also takes a device int64 tensor for
    ``performed`` (the op API's meters are computed on the GPU): it is kept on the device and resolved,
    with one host read for everything pending, only when ``performed`` is read -- the operators
    themselves never synchronise the host for the meter."""

    def __init__(self, performed: int = 0, dense_equiv: int = 0):
        self._performed = int(performed)
        self._pending = []
        self.dense_equiv = int(dense_equiv)

    @property
    def performed(self) -> int:
        if self._pending:
            self._performed += int(torch.stack([t.reshape(()) for t in self._pending]).sum().item())
            self._pending = []
        return self._performed

    @performed.setter
    def performed(self, v: int) -> None:
        self._performed, self._pending = int(v), []

    def add(self, performed, dense_equiv: int) -> None:
        if isinstance(performed, torch.Tensor):
            self._pending.append(performed.to(torch.int64))
        else:
            self._performed += int(performed)
        self.dense_equiv += int(dense_equiv)

    def reset(self) -> None:
        self.performed = 0
        self.dense_equiv = 0

    def snapshot(self):
        return self.performed, self.dense_equiv

    def __eq__(self, other):
        return isinstance(other, FlopCounter) and self.snapshot() == other.snapshot()

    def __repr__(self):
        return f"FlopCounter(performed={self.performed}, dense_equiv={self.dense_equiv})"


def _zeros_incr(shape, tile: TileShape, device):
    v = torch.zeros(shape, dtype=torch.float32, device=device)
    f = torch.zeros(grid_shape(shape, tile), dtype=torch.uint8, device=device)
    return v, f


def _desc(v, f, tile):
    c, h, w = v.shape
    return _lib.tdesc(_lib.ptr(v), _lib.ptr(f), 0, 0, c, h, w, tile.h, tile.w)


SPARSE_TILE_PATH_BELOW = 0.012  # live-tile fraction under which inc_conv2d gathers tiles
SCATTER_PATH_BELOW = float(os.environ.get("EVC_SCATTER_BELOW", "0.15"))  # input-stationary path below this (C4 sweep: scatter 329 vs fused 391 us at 10 %, 436 vs 393 at 20 %)


def inc_conv2d(x: IncrementTensor, weight, params: ConvParams, meter: FlopCounter) -> IncrementTensor:
    """Tile-skipping sparse convolution of an increment, bias dropped (increment_ops.py:126-194)."""
    dev = x.values.device
    weight = as_matrix(weight, dev)
    c_out, c_in, kh, kw = tuple(weight.shape)
    if tuple(params.kernel) != (kh, kw) or params.c_in != c_in or params.c_out != c_out:
        raise ValueError(f"weight shape {tuple(weight.shape)} disagrees with {params}")
    c, h, w = x.shape
    if c != c_in:
        raise ValueError(f"increment has {c} channels but conv expects {c_in}")
    st, pad = params.stride, params.padding
    ho, wo = conv_output_hw(h, w, kh, kw, st, pad)
    tile = x.tile
    meter.add(0, 2 * kh * kw * c_in * c_out * ho * wo)
    lib = _lib.lib()
    # very sparse increments: the gathered-tile GEMM touches only the active 6x6 output tiles,
    # while the fused kernel computes whole 128-site regions around them (measured on C4,
    # 64 -> 128 @ 480x640: 252 vs 398 us at 0.5 % live tiles; the fused path wins from ~1.5 %)
    kernel = None
    live = 1.0 - x.mask.false_fraction() if tensors.CONV_KERNEL == "tc" else 1.0
    plan = tensors.cached_plan(weight, st, pad, h, w, tile.h, tile.w)
    scatter = (tensors.CONV_KERNEL == "tc" and plan.path == "fused" and live < SCATTER_PATH_BELOW
               and plan.scatter_plan() is not None)
    if not scatter and tensors.CONV_KERNEL == "tc" and live < SPARSE_TILE_PATH_BELOW:
        kernel = "tile"
        plan = tensors.cached_plan(weight, st, pad, h, w, tile.h, tile.w, kernel=kernel)
    yv, yf = _zeros_incr((c_out, ho, wo), tile, dev)
    s = _lib.stream_ptr()
    din = x.desc()
    dout = _desc(yv, yf, tile)
    if scatter:
        # sparse increments: input-stationary gather -> GEMM -> scatter-add over the live input tiles
        # only (the meter's own unit of work); output flags and meter from the mask kernel
        i32 = torch.zeros(1, dtype=torch.int32, device=dev)
        scratch = torch.zeros(int(lib.evc_conv_mask_scratch(plan.g, 1)), dtype=torch.int32, device=dev)
        perf = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(lib.evc_conv_mask(*plan.mask_args(din, dout, _lib.ptr(scratch), _lib.ptr(i32), None, None,
                                                     _lib.ptr(perf)), s), "conv_mask")
        fn, args = plan.scatter(din, dout, fresh_out=True)
        _lib.check(fn(*args, s), "conv_scatter")
        meter.add(perf, 0)
        return IncrementTensor(yv, TileMask(yf, tile))
    if plan.path == "fused":
        fany = torch.zeros(plan.gi[0] * plan.gi[1], dtype=torch.uint8, device=dev)
        mpart = torch.zeros(plan.ctas * 2, dtype=torch.int64, device=dev)  # per-CTA meter partials
        _lib.check(lib.evc_tile_any(din, _lib.ptr(fany), 1, s), "tile_any")
        pre = plan.prep(din)
        _lib.check(pre[0](*pre[1], s), "to_hwc")
        fn, args = plan.fused(din, dout, fany=_lib.ptr(fany), mpart=_lib.ptr(mpart))
        _lib.check(fn(*args, s), "conv_fused")
        # performed (increment_ops.py:145-160): 0 when no input flag is live, the dense count when all are,
        # else 2 * C_out * the weighted live-tap term -- on the device, no host read
        cb = mpart.view(-1, 2).sum(dim=0)
        n_flags = c_in * plan.gi[0] * plan.gi[1]
        perf = torch.where(cb[0] == 0, torch.zeros_like(cb[1]),
                           torch.where(cb[0] == n_flags, torch.full_like(cb[1], int(plan.dense_flops)), 2 * c_out * cb[1]))
        meter.add(perf, 0)
        return IncrementTensor(yv, TileMask(yf, tile))
    T = yf.shape[1] * yf.shape[2]
    i32 = torch.zeros(2, dtype=torch.int32, device=dev)  # [in_true, tile_count]
    tiles = torch.empty(T, dtype=torch.int32, device=dev)
    scratch = torch.zeros(int(lib.evc_conv_mask_scratch(plan.g, 1)), dtype=torch.int32, device=dev)
    perf = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(lib.evc_conv_mask(*plan.mask_args(din, dout, _lib.ptr(scratch), _lib.ptr(i32), _lib.ptr(tiles),
                                                 _lib.ptr(i32) + 4, _lib.ptr(perf)), s), "conv_mask")
    ws = torch.empty(max(plan.ws_floats, 1), dtype=torch.float32, device=dev)
    fn, args = plan.gemm(din, dout, None, (_lib.ptr(tiles), _lib.ptr(i32) + 4), ws.data_ptr())
    _lib.check(fn(*args, s), "conv_gemm")
    meter.add(perf, 0)
    return IncrementTensor(yv, TileMask(yf, tile))


def flatten_increment(x: IncrementTensor) -> IncrementTensor:
    """Ravel to (1, 1, L) with a run-of-(h*w)-elements tile mask (increment_ops.py:197-202)."""
    run = x.tile.h * x.tile.w
    flat = x.values.reshape(1, 1, -1)
    return IncrementTensor(flat, make_tile_mask(flat, TileShape(1, run)))


def inc_linear(x_flat: IncrementTensor, matrix, meter: FlopCounter) -> IncrementTensor:
    """Matrix application to a flattened increment, dead runs skipped (increment_ops.py:205-223)."""
    dev = x_flat.values.device
    matrix = as_matrix(matrix, dev)
    c, h, length = x_flat.shape
    if (c, h) != (1, 1):
        raise ValueError(f"inc_linear expects a (1, 1, L) increment, got {x_flat.shape}")
    rows, cols = matrix.shape
    if cols != length:
        raise ValueError(f"matrix {tuple(matrix.shape)} does not apply to increment of length {length}")
    meter.add(0, 2 * rows * cols)
    tile = x_flat.tile
    out_shape = (1, 1, rows)
    y = torch.empty(rows, dtype=torch.float32, device=dev)
    lib = _lib.lib()
    ws = torch.empty(int(lib.evc_linear_workspace(rows, length, tile.h * tile.w, 1)), dtype=torch.float32,
                     device=dev)
    perf = torch.zeros(1, dtype=torch.int64, device=dev)
    din = _lib.tdesc(_lib.ptr(x_flat.values), _lib.ptr(x_flat.mask.u8), 0, 0, 1, 1, length, tile.h, tile.w)
    dout = _lib.tdesc(_lib.ptr(y), None, 0, 0, rows, 1, 1, 1, 1)
    _lib.check(lib.evc_linear(din, _lib.ptr(matrix), None, dout, rows, 0, _lib.ptr(perf), _lib.ptr(ws), 1,
                              _lib.stream_ptr()), "linear")
    meter.add(perf, 0)
    flags = torch.ones(grid_shape(out_shape, tile), dtype=torch.uint8, device=dev)
    return IncrementTensor(y.reshape(out_shape), TileMask(flags, tile))


def inc_add(a: IncrementTensor, b: IncrementTensor) -> IncrementTensor:
    """increment_ops.py:226-229."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.tile != b.tile:
        raise ValueError(f"tile shape mismatch: {a.tile} vs {b.tile}")
    yv, yf = _zeros_incr(a.shape, a.tile, a.values.device)
    _lib.check(_lib.lib().evc_add(a.desc(), b.desc(), _desc(yv, yf, a.tile), 1, _lib.stream_ptr()), "add")
    return IncrementTensor(yv, TileMask(yf, a.tile))


def _act(fn) -> Activation:
    if isinstance(fn, Activation):
        return fn
    if isinstance(fn, str):
        return Activation(fn)
    raise ValueError(f"activation must come from resolve_activation, got {fn!r}")


def inc_activation(x: IncrementTensor, state: AccState, fn) -> IncrementTensor:
    """f(acc + dx) - f(acc), then acc += dx (increment_ops.py:232-238)."""
    if tuple(state.x_acc.shape) != x.shape:
        raise ValueError(f"accumulator shape {tuple(state.x_acc.shape)} vs increment {x.shape}")
    f = _act(fn)
    yv, yf = _zeros_incr(x.shape, x.tile, x.values.device)
    _lib.check(_lib.lib().evc_act_delta(x.desc(), _lib.ptr(state.x_acc), 0, _desc(yv, yf, x.tile), f.code, f.alpha, 1,
                                        _lib.stream_ptr()), "act_delta")
    return IncrementTensor(yv, TileMask(yf, x.tile))


def inc_mul(a: IncrementTensor, b: IncrementTensor, sa: AccState, sb: AccState) -> IncrementTensor:
    """(acc_a + a) * b + acc_b * a; both accumulators fold (increment_ops.py:241-254)."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.tile != b.tile:
        raise ValueError(f"tile shape mismatch: {a.tile} vs {b.tile}")
    yv, yf = _zeros_incr(a.shape, a.tile, a.values.device)
    _lib.check(_lib.lib().evc_mul(a.desc(), b.desc(), _lib.ptr(sa.x_acc), _lib.ptr(sb.x_acc), 0,
                                  _desc(yv, yf, a.tile), 1, _lib.stream_ptr()), "mul")
    return IncrementTensor(yv, TileMask(yf, a.tile))


def inc_concat(parts) -> IncrementTensor:
    """Channel concatenation of values and masks (increment_ops.py:257-268)."""
    if not parts:
        raise ValueError("concat of zero parts")
    first = parts[0]
    for p in parts[1:]:
        if p.shape[1:] != first.shape[1:]:
            raise ValueError(f"spatial mismatch in concat: {p.shape} vs {first.shape}")
        if p.tile != first.tile:
            raise ValueError(f"tile mismatch in concat: {p.tile} vs {first.tile}")
    values = torch.cat([p.values for p in parts], dim=0)
    flags = torch.cat([p.mask.u8 for p in parts], dim=0)
    return IncrementTensor(values, TileMask(flags, first.tile))


def inc_upsample(x: IncrementTensor, factor: int, mode: str = "nearest") -> IncrementTensor:
    """Linear upsampling of the increment; mask follows the support (increment_ops.py:271-285)."""
    if factor not in (2, 4):
        raise ValueError(f"upsample factor must be 2 or 4, got {factor}")
    if mode not in ("nearest", "bilinear"):
        raise ValueError(f"unknown upsample mode {mode!r}")
    c, h, w = x.shape
    yv, yf = _zeros_incr((c, h * factor, w * factor), x.tile, x.values.device)
    _lib.check(_lib.lib().evc_upsample(x.desc(), _desc(yv, yf, x.tile), factor, 0 if mode == "nearest" else 1, 1,
                                       _lib.stream_ptr()), "upsample")
    return IncrementTensor(yv, TileMask(yf, x.tile))


def inc_maxpool(x: IncrementTensor, state: AccState, window=(2, 2), stride: int = 2) -> IncrementTensor:
    """maxpool(acc + dx) - maxpool(acc), then acc += dx (increment_ops.py:288-310)."""
    if tuple(state.x_acc.shape) != x.shape:
        raise ValueError(f"accumulator shape {tuple(state.x_acc.shape)} vs increment {x.shape}")
    c, h, w = x.shape
    wh, ww = window
    if wh > h or ww > w:
        raise ValueError(f"pool window {wh}x{ww} larger than input {h}x{w}")
    ho, wo = (h - wh) // stride + 1, (w - ww) // stride + 1
    yv, yf = _zeros_incr((c, ho, wo), x.tile, x.values.device)
    _lib.check(_lib.lib().evc_maxpool(x.desc(), _lib.ptr(state.x_acc), 0, _desc(yv, yf, x.tile), wh, ww, stride, 1,
                                      _lib.stream_ptr()), "maxpool")
    return IncrementTensor(yv, TileMask(yf, x.tile))
