"""Device tensors, tile masks and the dense operators (mirrors evincr/tensors.py).

All activations are float32 CUDA tensors of shape (C, H, W), channel-planar
like the reference (tensors.py:1-6).  A TileMask holds a per-channel uint8
grid (C, ceil(H/h), ceil(W/w)) on the device; ``.flags`` exposes it as a
bool view, the reference's dtype.  Numpy inputs are accepted at the edges
and uploaded.  Every operator runs in libevconv.so; there is no CPU path.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "TileShape",
    "TileMask",
    "IncrementTensor",
    "as_tensor",
    "grid_shape",
    "make_tile_mask",
    "all_true_mask",
    "all_false_mask",
    "mask_or",
    "mask_to_pixels",
    "integrate",
    "conv_output_hw",
    "dense_conv2d",
    "dense_linear",
    "dense_maxpool",
    "dense_upsample",
    "resolve_activation",
]

DEFAULT_TILE = (6, 6)
DEV = "cuda"


def _dev():
    _lib.lib()
    return torch.device(DEV, torch.cuda.current_device())


def as_tensor(data) -> torch.Tensor:
    """Coerce to a contiguous float32 (C, H, W) CUDA tensor (tensors.py:39-44)."""
    if isinstance(data, torch.Tensor):
        t = data.to(device=_dev(), dtype=torch.float32).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32)).to(_dev())
    if t.dim() != 3:
        raise ValueError(f"expected a 3-D (C, H, W) tensor, got shape {tuple(t.shape)}")
    return t


@dataclass(frozen=True)
class TileShape:
    """Spatial extent of one mask tile, in pixels (tensors.py:47-56)."""

    h: int = DEFAULT_TILE[0]
    w: int = DEFAULT_TILE[1]

    def __post_init__(self):
        if self.h < 1 or self.w < 1:
            raise ValueError(f"tile sides must be >= 1, got {self.h}x{self.w}")


def grid_shape(shape, tile: TileShape):
    """(C, ceil(H/h), ceil(W/w)) (tensors.py:59-62)."""
    c, h, w = shape
    return int(c), -(-int(h) // tile.h), -(-int(w) // tile.w)


def _as_flags(flags) -> torch.Tensor:
    if isinstance(flags, torch.Tensor):
        f = flags.to(_dev())
        if f.dtype == torch.bool:
            f = f.view(torch.uint8)
        elif f.dtype != torch.uint8:
            f = (f != 0).view(torch.uint8)
        return f.contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(flags, dtype=bool)).view(np.uint8)).to(_dev())


class TileMask:
    """Per-channel tile grid; False marks a tile known to be all-zero (tensors.py:65-90)."""

    __slots__ = ("_u8", "tile")

    def __init__(self, flags, tile: TileShape = None):
        u8 = _as_flags(flags)
        if u8.dim() != 3:
            raise ValueError(f"mask grid must be 3-D (C, gh, gw), got {tuple(u8.shape)}")
        self._u8 = u8
        self.tile = tile if tile is not None else TileShape()

    @property
    def flags(self) -> torch.Tensor:
        return self._u8.view(torch.bool)

    @property
    def u8(self) -> torch.Tensor:
        return self._u8

    @property
    def grid(self):
        return tuple(self._u8.shape)

    def false_fraction(self) -> float:
        n = self._u8.numel()
        return float(1.0 - int(self._u8.sum().item()) / n) if n else 0.0

    def covers(self, shape) -> bool:
        return self.grid == grid_shape(shape, self.tile)

    def active_indices(self) -> torch.Tensor:
        """Sorted active tile list == np.flatnonzero(flags), computed on device
        by warp-ballot compaction (evc_compact)."""
        n = self._u8.numel()
        idx = torch.empty(max(n, 1), dtype=torch.int32, device=self._u8.device)
        cnt = torch.zeros(1, dtype=torch.int32, device=self._u8.device)
        scratch = torch.empty(int(_lib.lib().evc_compact_scratch(n)), dtype=torch.int32, device=self._u8.device)
        _lib.check(_lib.lib().evc_compact(_lib.ptr(self._u8), n, _lib.ptr(idx), _lib.ptr(cnt), _lib.ptr(scratch),
                                          _lib.stream_ptr()), "compact")
        return idx[: int(cnt.item())].to(torch.int64)

    def numpy(self) -> np.ndarray:
        return self._u8.cpu().numpy().astype(bool)


class IncrementTensor:
    """Step-to-step difference tensor paired with a sound tile mask (tensors.py:133-164)."""

    __slots__ = ("values", "mask")

    def __init__(self, values, mask: TileMask):
        self.values = as_tensor(values)
        self.mask = mask
        if not mask.covers(tuple(self.values.shape)):
            raise ValueError(
                f"mask grid {mask.grid} does not cover tensor {tuple(self.values.shape)} "
                f"at tile {mask.tile.h}x{mask.tile.w}")

    @property
    def shape(self):
        return tuple(self.values.shape)

    @property
    def tile(self) -> TileShape:
        return self.mask.tile

    @classmethod
    def from_dense(cls, values, tile: TileShape) -> "IncrementTensor":
        values = as_tensor(values)
        return cls(values, make_tile_mask(values, tile))

    @classmethod
    def zeros(cls, shape, tile: TileShape) -> "IncrementTensor":
        return cls(torch.zeros(shape, dtype=torch.float32, device=_dev()), all_false_mask(shape, tile))

    def desc(self) -> _lib.EvcTensor:
        c, h, w = self.shape
        return _lib.tdesc(_lib.ptr(self.values), _lib.ptr(self.mask.u8), 0, 0, c, h, w, self.tile.h, self.tile.w)


def make_tile_mask(t, tile: TileShape) -> TileMask:
    """Exact mask: a tile is True iff it holds a nonzero (tensors.py:93-107)."""
    t = as_tensor(t)
    c, h, w = t.shape
    flags = torch.empty(grid_shape((c, h, w), tile), dtype=torch.uint8, device=t.device)
    d = _lib.tdesc(_lib.ptr(t), _lib.ptr(flags), 0, 0, c, h, w, tile.h, tile.w)
    _lib.check(_lib.lib().evc_make_tile_mask(d, 1, _lib.stream_ptr()), "make_tile_mask")
    return TileMask(flags, tile)


def all_true_mask(shape, tile: TileShape) -> TileMask:
    return TileMask(torch.ones(grid_shape(shape, tile), dtype=torch.uint8, device=_dev()), tile)


def all_false_mask(shape, tile: TileShape) -> TileMask:
    return TileMask(torch.zeros(grid_shape(shape, tile), dtype=torch.uint8, device=_dev()), tile)


def mask_or(a: TileMask, b: TileMask) -> TileMask:
    """Elementwise OR over the same grid (tensors.py:118-124)."""
    if a.tile != b.tile:
        raise ValueError(f"tile shape mismatch: {a.tile} vs {b.tile}")
    if a.grid != b.grid:
        raise ValueError(f"mask grid mismatch: {a.grid} vs {b.grid}")
    return TileMask(a.u8 | b.u8, a.tile)


def mask_to_pixels(mask: TileMask, h: int, w: int) -> torch.Tensor:
    """Per-pixel bool (C, h, w) (tensors.py:127-130)."""
    px = mask.flags.repeat_interleave(mask.tile.h, dim=1).repeat_interleave(mask.tile.w, dim=2)
    return px[:, :h, :w]


def integrate(dense, incr: IncrementTensor) -> torch.Tensor:
    """dense + increment on live tiles (tensors.py:167-174)."""
    dense = as_tensor(dense)
    if tuple(dense.shape) != incr.shape:
        raise ValueError(f"shape mismatch: {tuple(dense.shape)} vs {incr.shape}")
    out = dense.clone()
    _lib.check(_lib.lib().evc_integrate(_lib.ptr(out), 0, incr.desc(), 1, _lib.stream_ptr()), "integrate")
    return out


# ---------------------------------------------------------------------------
# dense operators
# ---------------------------------------------------------------------------


def conv_output_hw(h: int, w: int, kh: int, kw: int, stride: int, padding: int):
    """tensors.py:194-202."""
    h_out = (h + 2 * padding - kh) // stride + 1
    w_out = (w + 2 * padding - kw) // stride + 1
    if h_out < 1 or w_out < 1:
        raise ValueError(
            f"kernel {kh}x{kw} with stride {stride}, padding {padding} does not fit a {h}x{w} input")
    return h_out, w_out


_TABLES: dict = {}


def conv_geometry(c_in, c_out, kh, kw, stride, pad, h, w, th, tw):
    """(EvcConvGeom, device int32 table) for one conv layer, cached."""
    key = (c_in, c_out, kh, kw, stride, pad, h, w, th, tw, torch.cuda.current_device())
    hit = _TABLES.get(key)
    if hit is not None:
        return hit
    ho, wo = conv_output_hw(h, w, kh, kw, stride, pad)
    g = _lib.EvcConvGeom(c_in, c_out, kh, kw, stride, pad, h, w, ho, wo, th, tw)
    lib = _lib.lib()
    n = int(lib.evc_conv_table_len(g))
    host = np.zeros(n, dtype=np.int32)
    _lib.check(lib.evc_conv_table_fill(g, host.ctypes.data), "conv_table_fill")
    tab = torch.from_numpy(host).to(_dev())
    _TABLES[key] = (g, tab)
    return g, tab


CONV_KERNEL = os.environ.get("EVC_CONV_KERNEL", "tc")  # "tc" (tcgen05 3xTF32), "tile" (gathered tiles only), "simt"
# Sub-pixel decoder convs (ConvPlan._init_subpixel; the Graph's policy: graph.SUBPIXEL_MIN_SESSIONS,
# EVC_SUBPIXEL) only for thin decoder convs: with C_out > 32 the composed conv (4 x C_out channels on
# the low-res grid) was no faster than the high-res one even in isolation (scripts/conv_bench.py).
SUBPIXEL_MAX_COUT = int(os.environ.get("EVC_SUBPIXEL_MAX_COUT", "32"))


def pack_conv_weight(weight: torch.Tensor):
    """Pre-split (hi/lo) + 128B-swizzle a (C_out, C_in, KH, KW) weight for the tcgen05 kernel."""
    c_out = int(weight.shape[0])
    k = int(np.prod(weight.shape[1:]))
    lib = _lib.lib()
    host = np.ascontiguousarray(weight.detach().cpu().numpy().reshape(c_out, k), dtype=np.float32)
    out = np.zeros(int(lib.evc_conv_tc_pack_len(c_out, k)), dtype=np.float32)
    _lib.check(lib.evc_conv_tc_pack(host.ctypes.data, c_out, k, out.ctypes.data), "conv_tc_pack")
    return torch.from_numpy(out).to(weight.device)


_PLANS: dict = {}


def cached_plan(weight: torch.Tensor, stride, pad, h, w, th, tw, kernel: str | None = None) -> "ConvPlan":
    """ConvPlan for the stateless op API (inc_conv2d / dense_conv2d), cached per weight tensor
    and geometry: the weight packing, tables and shadow buffer are built once, not per call.
    The key holds the tensor's data pointer and version counter, so an in-place update of the
    weights (or a new tensor) gets a fresh plan; the dense kernel kind is part of the key."""
    kernel = kernel or CONV_KERNEL
    key = (weight.data_ptr(), weight._version, tuple(weight.shape), str(weight.device), int(stride), int(pad),
           int(h), int(w), int(th), int(tw), kernel)
    plan = _PLANS.get(key)
    if plan is None:
        if len(_PLANS) >= 8:  # each plan holds its shadow buffer
            _PLANS.clear()
        plan = ConvPlan(weight, stride, pad, h, w, th, tw, kernel=kernel)
        _PLANS[key] = plan
    return plan


class ConvPlan:
    """Static launch plan of one conv layer: geometry table, kernel path, packed weights, K-splits.

    path "fused": TMA-fed tcgen05 GEMM over live RH x RW output regions with the mask
    propagation, the FLOP meter, the split-K reduction (thread-block cluster) and an
    optional activation delta in the same launch (evc_conv_fused); path "tile": tcgen05
    GEMM over gathered sites of the active 6x6 output tiles after evc_conv_mask (geometries
    the fused kernel does not take: padding >= kernel); path "simt": FFMA reference kernel.
    """

    def __init__(self, weight: torch.Tensor, stride, pad, h, w, th, tw, S=1, vstride=None, kernel=None,
                 max_splits: int = 0, subpixel: bool = False):
        lib = _lib.lib()
        c_out, c_in, kh, kw = (int(v) for v in weight.shape)
        self.g, self.table = conv_geometry(c_in, c_out, kh, kw, stride, pad, h, w, th, tw)
        self.subpixel = False
        if subpixel:  # (the Graph checked subpixel_ok: the input is a 2x bilinear upsample)
            self._init_subpixel(weight, h, w, th, tw, S, max_splits)
            return
        self.c_out, self.c_in, self.kh, self.kw, self.S = c_out, c_in, kh, kw, S
        self.weight = weight
        kernel = kernel or CONV_KERNEL
        ho, wo = int(self.g.Ho), int(self.g.Wo)
        T = -(-ho // th) * -(-wo // tw)
        self.T = T
        self.wpack = None
        self.hwc = None
        self.fed_by_sparsify = False  # set by the Graph: a sparsify writes this conv's input shadow
        self.gi = (-(-h // th), -(-w // tw))  # input tile grid
        if kernel == "tc" and lib.evc_conv_fused_supported(self.g):
            self.path = "fused"
            self.cfg = _lib.EvcConvCfg()
            _lib.check(lib.evc_conv_fused_config(self.g, S, int(max_splits), self.cfg), "conv_fused_config")
            # channels per shadow pixel: 32-aligned for the TMA path, 4-aligned for the CUDA-core path
            self.cp = -(-c_in // 4) * 4 if self.cfg.thin else int(lib.evc_hwc_channels(c_in))
            # the CUDA-core path reads plain fp32 values (cp < 0 at the ABI, common.cuh hwc_px);
            # the tensor-core path the hi/lo split
            self.cpa = -self.cp if self.cfg.thin else self.cp
            self.px = self.cp if self.cfg.thin else 2 * self.cp
            # shadow with a zero border of the conv's padding: (S, H + 2p, W + 2p, px)
            self.pitch = w + 2 * pad
            self.hwc = torch.zeros((S, h + 2 * pad, self.pitch, self.px), dtype=torch.float32,
                                   device=weight.device)
            self.hwc_interior = self.hwc.data_ptr() + 4 * (pad * self.pitch + pad) * self.px
            host = np.ascontiguousarray(weight.detach().cpu().numpy(), dtype=np.float32)
            out = np.zeros(int(lib.evc_conv_fused_pack_len(self.g, self.cfg)), dtype=np.float32)
            _lib.check(lib.evc_conv_fused_pack(host.ctypes.data, self.g, self.cfg, out.ctypes.data), "pack")
            self.wpack = torch.from_numpy(out).to(weight.device)
            self.rstate = torch.zeros(int(lib.evc_conv_fused_state_len(self.g, self.cfg, S)), dtype=torch.uint8,
                                      device=weight.device)
            self.splits = int(self.cfg.splits)
            self.ws_floats = 0
            self.ctas = int(lib.evc_conv_fused_ctas(self.g, self.cfg))  # per session (meter partials)
        else:
            self.path = "tile" if kernel in ("tc", "tile") else "simt"
            if self.path == "tile":
                self.wpack = pack_conv_weight(weight)
            self.splits = choose_splits(S * T * th * tw, c_out, c_in * kh * kw, kernel=kernel)
            self.ws_floats = int(lib.evc_conv_workspace(self.g, S * T, self.splits))
        self.dense_flops = 2 * kh * kw * c_in * c_out * ho * wo

    @staticmethod
    def subpixel_ok(weight, stride, pad, h, w) -> bool:
        """Whether a conv fed by a 2x bilinear upsample can run in sub-pixel form."""
        c_out, _, kh, kw = (int(v) for v in weight.shape)
        return (kh == kw == 3 and stride == 1 and pad == 1 and c_out % 4 == 0 and h % 2 == 0 and w % 2 == 0
                and c_out <= SUBPIXEL_MAX_COUT and CONV_KERNEL == "tc")

    def _init_subpixel(self, weight, h, w, th, tw, S, max_splits):
        """Sub-pixel plan (csrc/subpixel.cu): the conv of the 2x bilinear upsample of a (C, h/2, w/2)
        input as ONE 3x3 conv of that low-res input with 4 x C_out composed channels (compose_subpixel),
        reading a low-res hi/lo shadow with a replicated edge ring (evc_subpixel_prep) plus a
        border-line correction (evc_subpixel_border).  self.table / flags / meter stay the real
        (high-res) conv's; self.g / cfg / wpack / rstate describe the composed launch."""
        lib = _lib.lib()
        c_out, c_in = int(weight.shape[0]), int(weight.shape[1])
        self.subpixel = True
        self.c_out, self.c_in, self.kh, self.kw, self.S = c_out, c_in, 3, 3, S
        self.weight = weight.contiguous()
        self.g_hi = self.g
        ho, wo = int(self.g.Ho), int(self.g.Wo)
        self.T = -(-ho // th) * -(-wo // tw)
        hl, wl = h // 2, w // 2
        self.g, _ = conv_geometry(c_in, 4 * c_out, 3, 3, 1, 1, hl, wl, th, tw)
        self.path = "fused"
        self.fed_by_sparsify = False
        self.gi = (-(-h // th), -(-w // tw))  # the real conv's input tile grid (fany of the sparsify)
        self.cfg = _lib.EvcConvCfg()
        _lib.check(lib.evc_conv_fused_config(self.g, S, int(max_splits), self.cfg), "conv_fused_config")
        self.cp = int(lib.evc_hwc_channels(c_in))
        self.cpa, self.px = self.cp, 2 * self.cp
        self.pitch = wl + 2
        self.hwc = torch.zeros((S, hl + 2, self.pitch, self.px), dtype=torch.float32, device=weight.device)
        self.hwc_interior = self.hwc.data_ptr() + 4 * (self.pitch + 1) * self.px
        host = np.ascontiguousarray(compose_subpixel(weight.detach().cpu().numpy()), dtype=np.float32)
        out = np.zeros(int(lib.evc_conv_fused_pack_len(self.g, self.cfg)), dtype=np.float32)
        _lib.check(lib.evc_conv_fused_pack(host.ctypes.data, self.g, self.cfg, out.ctypes.data), "pack")
        self.wpack = torch.from_numpy(out).to(weight.device)
        self.rstate = torch.zeros(int(lib.evc_conv_fused_state_len(self.g, self.cfg, S)), dtype=torch.uint8,
                                  device=weight.device)
        self.splits = int(self.cfg.splits)
        self.ws_floats = 0
        self.ctas = int(lib.evc_conv_fused_ctas(self.g, self.cfg))
        self.gl = (-(-hl // th), -(-wl // tw))  # low-res tile grid: its any-map (per-step zeroed) is
        self.fany_lo_ptr = None                  # placed by the owner (Graph: the step's scratch arena)
        self.wborder = self.weight.permute(1, 2, 3, 0).contiguous()  # (C_in, 3, 3, C_out) for the border GEMM
        self.border = torch.zeros((S, 2 * (ho + wo), c_out), dtype=torch.float32, device=weight.device)
        self.dense_flops = 2 * 9 * c_in * c_out * ho * wo

    def subpixel_launches(self, dlo, dy, part_ptr, fany_hi):
        """[(fn, args-without-stream, name)] of the composed conv's inputs, from the low-res tensor dlo
        (the upsample's input): evc_subpixel_input (low-res shadow + tile map, and the sparsify's
        flags dy / any-map fany_hi / norm partials at part_ptr), evc_subpixel_border."""
        L = _lib.lib()
        # EVC_SUBPIX_FUSED=1: both passes in one launch (evc_subpixel_input_border) -- measured slower at 32
        # streams (621 vs 423 + 177 us per step), so two launches by default
        if os.environ.get("EVC_SUBPIX_FUSED") == "1":
            return [(L.evc_subpixel_input_border, (dlo, dy, part_ptr, self.hwc_interior, self.cp, self.hwc[0].numel(),
                                                   self.pitch, self.fany_lo_ptr, fany_hi, self.wborder.data_ptr(),
                                                   self.c_out, self.border.data_ptr(), self.S), "subpixel_input_border")]
        return [(L.evc_subpixel_input, (dlo, dy, part_ptr, self.hwc_interior, self.cp, self.hwc[0].numel(),
                                        self.pitch, self.fany_lo_ptr, fany_hi, self.S), "subpixel_input"),
                (L.evc_subpixel_border, (dlo, self.wborder.data_ptr(), self.c_out, self.border.data_ptr(), self.S),
                 "subpixel_border")]

    def scatter_plan(self):
        """Packed weights + workspace of the input-stationary scatter path (evc_conv_scatter) for
        this layer, built on first use; None when the geometry is not supported."""
        sp = getattr(self, "_scatter", None)
        if sp is None:
            lib = _lib.lib()
            if not lib.evc_conv_scatter_supported(self.g):
                self._scatter = False
                return None
            host = np.ascontiguousarray(self.weight.detach().cpu().numpy(), dtype=np.float32)
            out = np.zeros(int(lib.evc_conv_scatter_pack_len(self.g)), dtype=np.float32)
            _lib.check(lib.evc_conv_scatter_pack(host.ctypes.data, self.g, out.ctypes.data), "scatter_pack")
            ws = torch.zeros(int(lib.evc_conv_scatter_workspace(self.g, self.S)), dtype=torch.uint8,
                             device=self.weight.device)
            sp = self._scatter = (torch.from_numpy(out).to(self.weight.device), ws)
        return sp or None

    def scatter(self, din, dout, fresh_out: bool):
        """(ctypes fn, args-without-stream) of evc_conv_scatter (values only)."""
        wp, ws = self.scatter_plan()
        return _lib.lib().evc_conv_scatter, (self.g, din, wp.data_ptr(), dout, ws.data_ptr(), ws.numel(),
                                             1 if fresh_out else 0, self.S)

    def prep(self, din):
        """(fn, args-without-stream) mirroring the conv input into the HWC shadow, or None."""
        if self.path != "fused":
            return None
        return _lib.lib().evc_to_hwc, (din, self.hwc_interior, self.hwc[0].numel(), self.cpa, self.pitch, self.S)

    def mask_args(self, din, dout, scratch, in_true, tile_list, tile_count, meter):
        """evc_conv_mask arguments of the unfused paths (stream appended by the caller)."""
        return (self.g, din, dout, self.table.data_ptr(), scratch, in_true, tile_list, tile_count, None, meter,
                self.S)

    def fused(self, din, dout, *, fany=None, mpart=None, bias_ptr=None, act=None, sp=None, dense=False):
        """(ctypes fn, args-without-stream) of evc_conv_fused.

        act = (code, alpha, acc_ptr, acc_stride, act_desc) fuses the activation node;
        dout may then be None (conv values not materialised).  sp = EvcConvSparsify fuses
        the following t_p = 0 sparsify (the act desc may then carry no values)."""
        code, alpha, acc, accs, adesc = act if act is not None else (-1, 0.0, None, 0, None)
        if self.subpixel:
            sub = _lib.EvcConvSubpixel(self.c_out, int(self.g_hi.Ho), int(self.g_hi.Wo), 0, fany,
                                       self.border.data_ptr())
            self._sub_keep = getattr(self, "_sub_keep", []) + [sub]  # alive as long as the program
            return _lib.lib().evc_conv_fused_subpixel, (self.g, self.cfg, self.hwc.data_ptr(), self.cpa,
                                                        self.hwc[0].numel(), self.wpack.data_ptr(), bias_ptr, din,
                                                        self.fany_lo_ptr, self.table.data_ptr(),
                                                        self.rstate.data_ptr(), mpart, dout, code, alpha, acc, accs,
                                                        adesc, sp, sub, 1 if dense else 0, self.S)
        return _lib.lib().evc_conv_fused, (self.g, self.cfg, self.hwc.data_ptr(), self.cpa, self.hwc[0].numel(),
                                           self.wpack.data_ptr(), bias_ptr, din, fany, self.table.data_ptr(),
                                           self.rstate.data_ptr(), mpart, dout, code, alpha, acc, accs,
                                           adesc, sp, 1 if dense else 0, self.S)

    def gemm(self, din, dout, bias_ptr, work, ws_ptr):
        """(ctypes fn, args-without-stream) of the unfused GEMM launch (tile / simt paths).

        work = None for the dense pass (every tile), else the (tile_list, tile_count)
        device pointers from conv_mask."""
        lib = _lib.lib()
        tl, tc = work if work is not None else (None, None)
        return lib.evc_conv_gemm, (self.g, din, self.weight.data_ptr(), _lib.ptr(self.wpack), bias_ptr, dout,
                                   self.table.data_ptr(), tl, tc, self.S, self.splits, ws_ptr)


# half-pixel 2x bilinear taps per output phase: _SUBPIX_TAPS[a][d + 1][k] = weight of low-res offset
# d in the upsampled value that kernel tap k of a 3x3 conv reads for output phase a (tensors.py:259-266)
_SUBPIX_TAPS = np.zeros((2, 3, 3))
_SUBPIX_TAPS[0, 0, 0], _SUBPIX_TAPS[0, 1, 0] = 0.75, 0.25
_SUBPIX_TAPS[0, 0, 1], _SUBPIX_TAPS[0, 1, 1] = 0.25, 0.75
_SUBPIX_TAPS[0, 1, 2], _SUBPIX_TAPS[0, 2, 2] = 0.75, 0.25
_SUBPIX_TAPS[1, 0, 0], _SUBPIX_TAPS[1, 1, 0] = 0.25, 0.75
_SUBPIX_TAPS[1, 1, 1], _SUBPIX_TAPS[1, 2, 1] = 0.75, 0.25
_SUBPIX_TAPS[1, 1, 2], _SUBPIX_TAPS[1, 2, 2] = 0.25, 0.75


def compose_subpixel(weight) -> np.ndarray:
    """(4 C_out, C_in, 3, 3) weights of the sub-pixel conv: composed channel 4 o + 2 a + b (phase-minor)
    is output channel o at phase (a, b) (site (2i + a, 2j + b)) of conv3x3(upsample2x_bilinear(x)),
    evaluated on x itself (edge-replicated).  Composed in float64, rounded once."""
    w = np.asarray(weight, dtype=np.float64)
    co = w.shape[0]
    out = np.zeros((4 * co, *w.shape[1:]))
    for a in range(2):
        for b in range(2):
            out[2 * a + b::4] = np.einsum("yk,xl,oikl->oiyx", _SUBPIX_TAPS[a], _SUBPIX_TAPS[b], w)
    return out.astype(np.float32)


def choose_splits(max_sites: int, c_out: int, k: int, target_ctas: int = 2 * 148, kernel: str | None = None) -> int:
    """K-splits so the worst-case grid still fills the B200 (148 SMs)."""
    if (kernel or CONV_KERNEL) in ("tc", "tile"):
        ctas = max(1, -(-max_sites // 128)) * max(1, -(-c_out // 256))
        if ctas >= 148:
            return 1
        nkb = -(-k // 32)
        return int(max(1, min(-(-148 // ctas), nkb // 2, 64)))
    bm, bn = (128, 64) if c_out > 32 else ((128, 32) if c_out > 24 else (256, 16))
    ctas = max(1, -(-max_sites // bm)) * max(1, -(-c_out // bn))
    if ctas >= target_ctas:
        return 1
    s = -(-target_ctas // ctas)
    return int(max(1, min(s, k // 64, 32)))


def dense_conv2d(x, weight, bias=None, stride: int = 1, padding: int = 0) -> torch.Tensor:
    """Cross-correlation with zero padding and optional bias (tensors.py:205-228)."""
    x = as_tensor(x)
    weight = as_matrix(weight, x.device)
    if weight.dim() != 4:
        raise ValueError(f"weight must be (C_out, C_in, K_h, K_w), got {tuple(weight.shape)}")
    c_out, c_in, kh, kw = weight.shape
    c, h, w = x.shape
    if c != c_in:
        raise ValueError(f"input has {c} channels but weight expects {c_in}")
    ho, wo = conv_output_hw(h, w, kh, kw, stride, padding)
    th, tw = (4, 32) if wo >= 32 else (8, max(1, wo))
    plan = cached_plan(weight, stride, padding, h, w, th, tw)
    y = torch.empty((c_out, ho, wo), dtype=torch.float32, device=x.device)
    b = None if bias is None else as_bias(bias, c_out, x.device)
    din = _lib.tdesc(_lib.ptr(x), None, c * h * w, 0, c, h, w, th, tw)
    dout = _lib.tdesc(_lib.ptr(y), None, c_out * ho * wo, 0, c_out, ho, wo, th, tw)
    s = _lib.stream_ptr()
    if plan.path == "fused":
        pre = plan.prep(din)
        _lib.check(pre[0](*pre[1], s), "to_hwc")
        fn, args = plan.fused(din, dout, bias_ptr=_lib.ptr(b), dense=True)
        _lib.check(fn(*args, s), "conv_fused")
        return y
    ws = torch.empty(max(plan.ws_floats, 1), dtype=torch.float32, device=x.device)
    fn, args = plan.gemm(din, dout, _lib.ptr(b), None, ws.data_ptr())
    _lib.check(fn(*args, s), "conv_gemm")
    return y


def as_bias(bias, n, device):
    b = bias if isinstance(bias, torch.Tensor) else torch.from_numpy(np.asarray(bias, dtype=np.float32))
    return b.to(device=device, dtype=torch.float32).reshape(n).contiguous()


def as_matrix(m, device=None):
    t = m if isinstance(m, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(m, dtype=np.float32))
    return t.to(device=device or _dev(), dtype=torch.float32).contiguous()


def dense_linear(x_flat, matrix, bias=None) -> torch.Tensor:
    """matrix @ x (+ bias) (tensors.py:231-239)."""
    x = x_flat if isinstance(x_flat, torch.Tensor) else torch.from_numpy(np.asarray(x_flat, dtype=np.float32))
    x = x.to(_dev(), torch.float32).reshape(-1).contiguous()
    matrix = as_matrix(matrix, x.device)
    if matrix.dim() != 2 or matrix.shape[1] != x.shape[0]:
        raise ValueError(f"matrix {tuple(matrix.shape)} does not apply to vector of length {x.shape[0]}")
    f, length = matrix.shape
    y = torch.empty(f, dtype=torch.float32, device=x.device)
    b = None if bias is None else as_bias(bias, f, x.device)
    lib = _lib.lib()
    ws = torch.empty(int(lib.evc_linear_workspace(f, length, 1, 1)), dtype=torch.float32, device=x.device)
    din = _lib.tdesc(_lib.ptr(x), None, 0, 0, 1, 1, length, 1, 1)
    dout = _lib.tdesc(_lib.ptr(y), None, 0, 0, f, 1, 1, 1, 1)
    _lib.check(lib.evc_linear(din, _lib.ptr(matrix), _lib.ptr(b), dout, f, 1, None, _lib.ptr(ws), 1,
                              _lib.stream_ptr()), "linear")
    return y


def dense_maxpool(x, window=(2, 2), stride: int = 2) -> torch.Tensor:
    """No-padding max pooling (tensors.py:242-256)."""
    x = as_tensor(x)
    c, h, w = x.shape
    wh, ww = window
    if wh > h or ww > w:
        raise ValueError(f"pool window {wh}x{ww} larger than input {h}x{w}")
    ho, wo = (h - wh) // stride + 1, (w - ww) // stride + 1
    y = torch.empty((c, ho, wo), dtype=torch.float32, device=x.device)
    din = _lib.tdesc(_lib.ptr(x), None, 0, 0, c, h, w, 6, 6)
    dout = _lib.tdesc(_lib.ptr(y), None, 0, 0, c, ho, wo, 6, 6)
    _lib.check(_lib.lib().evc_maxpool(din, None, 0, dout, wh, ww, stride, 1, _lib.stream_ptr()), "maxpool")
    return y


def dense_upsample(x, factor: int, mode: str = "nearest") -> torch.Tensor:
    """Nearest / half-pixel bilinear upsampling (tensors.py:259-282)."""
    x = as_tensor(x)
    if factor not in (2, 4):
        raise ValueError(f"upsample factor must be 2 or 4, got {factor}")
    if mode not in ("nearest", "bilinear"):
        raise ValueError(f"unknown upsample mode {mode!r}")
    c, h, w = x.shape
    y = torch.empty((c, h * factor, w * factor), dtype=torch.float32, device=x.device)
    din = _lib.tdesc(_lib.ptr(x), None, 0, 0, c, h, w, 6, 6)
    dout = _lib.tdesc(_lib.ptr(y), None, 0, 0, c, h * factor, w * factor, 6, 6)
    _lib.check(_lib.lib().evc_upsample(din, dout, factor, 0 if mode == "nearest" else 1, 1, _lib.stream_ptr()),
               "upsample")
    return y


class Activation:
    """Elementwise activation f (tensors.py:285-312); callable on device tensors."""

    __slots__ = ("kind", "alpha", "code")

    def __init__(self, kind: str, alpha: float = 0.01):
        if kind not in _lib.ACT:
            raise ValueError(f"unknown activation {kind!r}")
        self.kind = kind
        self.alpha = float(np.float32(alpha))
        self.code = _lib.ACT[kind]

    def __call__(self, x):
        x = as_tensor(x)
        y = torch.empty_like(x)
        _lib.check(_lib.lib().evc_act_dense(_lib.ptr(x), 0, _lib.ptr(y), 0, None, 0, x.numel(), self.code,
                                            self.alpha, 1, _lib.stream_ptr()), "act_dense")
        return y

    def __repr__(self):
        return f"Activation({self.kind!r}, alpha={self.alpha})"


def resolve_activation(kind: str, alpha: float = 0.01) -> Activation:
    """Map an activation name to its elementwise function (tensors.py:303-312)."""
    return Activation(kind, alpha)
