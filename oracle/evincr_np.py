"""Numpy restatement of the reference ``evincr`` 0.1.0 incremental path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Every function
names the reference file:line it restates; paths are relative to
``/root/reference/pkg/src/evincr/``.

Representation: an increment is the pair ``(values, flags)`` where
``values`` is a float32 ``(C, H, W)`` array and ``flags`` a bool
``(C, ceil(H/th), ceil(W/tw))`` tile grid.  Accumulator / sparsifier
state lives in plain dicts so the restatement stays independent of the
product package.

Two convolution routes are provided:

* ``inc_conv2d``         -- values from one dense im2col GEMM of the
  increment (equal to the reference's per-channel sum up to float
  reassociation), masks from pixel liveness, FLOP meter from a vectorised
  live-tap count.  Fast; used by the tests as the checker.
* ``inc_conv2d_refalg``  -- the reference's own per-input-channel loop
  (``increment_ops.py:156-194``), kept so the CPU baseline in
  ``bench.py`` times the reference algorithm rather than a faster one.
"""

from __future__ import annotations

import heapq

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

F32 = np.float32

# ---------------------------------------------------------------------------
# tile masks  (tensors.py)
# ---------------------------------------------------------------------------


def tile_grid(shape, th, tw):
    """tensors.py:59-62 -- (C, ceil(H/th), ceil(W/tw))."""
    c, h, w = shape
    return c, (h + th - 1) // th, (w + tw - 1) // tw


def tile_flags(values, th, tw):
    """tensors.py:93-107 make_tile_mask: True iff the tile holds a nonzero
    (-0.0 counts as zero); boundary tiles cover the partial remainder."""
    v = np.asarray(values, dtype=F32)
    c, h, w = v.shape
    _, gh, gw = tile_grid(v.shape, th, tw)
    nz = np.zeros((c, gh * th, gw * tw), dtype=bool)
    nz[:, :h, :w] = v != 0
    return nz.reshape(c, gh, th, gw, tw).any(axis=(2, 4))


def tiles_any(px, th, tw):
    """increment_ops.py:116-123 _tiles_any over a boolean pixel map."""
    c, h, w = px.shape
    _, gh, gw = tile_grid(px.shape, th, tw)
    pad = np.zeros((c, gh * th, gw * tw), dtype=bool)
    pad[:, :h, :w] = px
    return pad.reshape(c, gh, th, gw, tw).any(axis=(2, 4))


def flags_to_pixels(flags, th, tw, h, w):
    """tensors.py:127-130 mask_to_pixels."""
    return np.repeat(np.repeat(flags, th, axis=1), tw, axis=2)[:, :h, :w]


def false_fraction(flags):
    """tensors.py:86-87 -- 1 - mean(flags) computed from the integer count."""
    n = flags.size
    return float(1.0 - np.count_nonzero(flags) / n) if n else 0.0


def active_index_list(flags):
    """The sorted active tile list: flatnonzero over (c, i, j) order."""
    return np.flatnonzero(np.asarray(flags).ravel()).astype(np.int64)


def integrate(dense, values, flags, th, tw):
    """tensors.py:167-174 -- dense + where(live_px, dx, 0)."""
    d = np.asarray(dense, dtype=F32)
    live = flags_to_pixels(flags, th, tw, d.shape[1], d.shape[2])
    return d + np.where(live, values, F32(0.0))


# ---------------------------------------------------------------------------
# dense operators  (tensors.py)
# ---------------------------------------------------------------------------


def conv_out_hw(h, w, kh, kw, stride, pad):
    """tensors.py:194-202."""
    ho = (h + 2 * pad - kh) // stride + 1
    wo = (w + 2 * pad - kw) // stride + 1
    if ho < 1 or wo < 1:
        raise ValueError(f"kernel {kh}x{kw} stride {stride} pad {pad} does not fit {h}x{w}")
    return ho, wo


def _patch_matrix(x, kh, kw, stride, pad, ho, wo):
    """(C*kh*kw, ho*wo) patch matrix, rows ordered (c, r, s) like tensors.py:182-191."""
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad))) if pad else x
    win = sliding_window_view(xp, (kh, kw), axis=(1, 2))  # (C, Hp-kh+1, Wp-kw+1, kh, kw)
    win = win[:, : stride * ho : stride, : stride * wo : stride]
    return np.ascontiguousarray(win.transpose(0, 3, 4, 1, 2)).reshape(-1, ho * wo)


def dense_conv2d(x, weight, bias=None, stride=1, pad=0):
    """tensors.py:205-228 -- cross-correlation, zero padding, optional bias."""
    x = np.asarray(x, dtype=F32)
    weight = np.asarray(weight, dtype=F32)
    co, ci, kh, kw = weight.shape
    c, h, w = x.shape
    if c != ci:
        raise ValueError(f"input has {c} channels but weight expects {ci}")
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    y = (weight.reshape(co, -1) @ _patch_matrix(x, kh, kw, stride, pad, ho, wo)).reshape(co, ho, wo)
    if bias is not None:
        y = y + np.asarray(bias, dtype=F32).reshape(co, 1, 1)
    return np.ascontiguousarray(y, dtype=F32)


def dense_linear(x_flat, matrix, bias=None):
    """tensors.py:231-239."""
    y = np.asarray(matrix, dtype=F32) @ np.asarray(x_flat, dtype=F32).reshape(-1)
    if bias is not None:
        y = y + np.asarray(bias, dtype=F32)
    return y.astype(F32)


def dense_maxpool(x, window=(2, 2), stride=2):
    """tensors.py:242-256 -- no padding."""
    x = np.asarray(x, dtype=F32)
    wh, ww = window
    _, h, w = x.shape
    if wh > h or ww > w:
        raise ValueError(f"pool window {wh}x{ww} larger than input {h}x{w}")
    ho, wo = (h - wh) // stride + 1, (w - ww) // stride + 1
    win = sliding_window_view(x, (wh, ww), axis=(1, 2))[:, : stride * ho : stride, : stride * wo : stride]
    return np.ascontiguousarray(win.max(axis=(3, 4)), dtype=F32)


def bilinear_taps(n_in, factor):
    """tensors.py:259-266 -- half-pixel source rows, clamped, float32 weights."""
    src = (np.arange(n_in * factor, dtype=F32) + F32(0.5)) / F32(factor) - F32(0.5)
    lo = np.floor(src).astype(np.int64)
    frac = (src - lo).astype(F32)
    hi = np.clip(lo + 1, 0, n_in - 1)
    lo = np.clip(lo, 0, n_in - 1)
    return lo, hi, frac


def dense_upsample(x, factor, mode="nearest"):
    """tensors.py:269-282 -- nearest repeat or separable bilinear (rows first)."""
    x = np.asarray(x, dtype=F32)
    if factor not in (2, 4):
        raise ValueError(f"upsample factor must be 2 or 4, got {factor}")
    if mode == "nearest":
        return np.ascontiguousarray(x.repeat(factor, axis=1).repeat(factor, axis=2))
    if mode != "bilinear":
        raise ValueError(f"unknown upsample mode {mode!r}")
    _, h, w = x.shape
    r0, r1, rf = bilinear_taps(h, factor)
    c0, c1, cf = bilinear_taps(w, factor)
    one = F32(1.0)
    rows = x[:, r0, :] * (one - rf)[None, :, None] + x[:, r1, :] * rf[None, :, None]
    out = rows[:, :, c0] * (one - cf)[None, None, :] + rows[:, :, c1] * cf[None, None, :]
    return np.ascontiguousarray(out, dtype=F32)


def activation(kind, alpha=0.01):
    """tensors.py:285-312 resolve_activation."""
    if kind == "relu":
        return lambda v: np.maximum(v, F32(0.0))
    if kind == "sigmoid":
        return lambda v: (1.0 / (1.0 + np.exp(-v))).astype(F32)
    if kind == "tanh":
        return lambda v: np.tanh(v).astype(F32)
    if kind == "leaky_relu":
        a = F32(alpha)
        return lambda v: np.where(v > 0, v, a * v).astype(F32)
    raise ValueError(f"unknown activation {kind!r}")


# ---------------------------------------------------------------------------
# increment operators  (increment_ops.py)
# ---------------------------------------------------------------------------


def conv_live_taps(flags, th, tw, h, w, kh, kw, stride, pad):
    """Per-channel live-tap counts L[c,u,v] and in-bounds tap counts inb[u,v].

    L counts the taps of output site (u, v) that land on a True tile of
    channel c (padding taps never count); inb counts all in-bounds taps.
    Together they give the reference meter (increment_ops.py:165-180).
    """
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    live = flags_to_pixels(flags, th, tw, h, w)
    livep = np.pad(live, ((0, 0), (pad, pad), (pad, pad))).astype(np.int32)
    inside = np.pad(np.ones((1, h, w), np.int32), ((0, 0), (pad, pad), (pad, pad)))
    L = np.zeros((flags.shape[0], ho, wo), np.int32)
    inb = np.zeros((1, ho, wo), np.int32)
    for r in range(kh):
        for s in range(kw):
            L += livep[:, r : r + stride * ho : stride, s : s + stride * wo : stride]
            inb += inside[:, r : r + stride * ho : stride, s : s + stride * wo : stride]
    return L, inb[0]


def conv_meter(flags, th, tw, h, w, c_out, kh, kw, stride, pad):
    """FLOP meter of inc_conv2d (increment_ops.py:144,148-154,180,191).

    Returns (performed, dense_equiv, active_any) where active_any is the
    per-output-pixel OR over channels of "some tap is live".
    """
    c_in = flags.shape[0]
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    kk = kh * kw
    dense = 2 * kk * c_in * c_out * ho * wo
    if not flags.any():
        return 0, dense, np.zeros((ho, wo), bool)
    if flags.all():
        return dense, dense, np.ones((ho, wo), bool)
    L, inb = conv_live_taps(flags, th, tw, h, w, kh, kw, stride, pad)
    run = L > 0
    per_site = np.where(run, kk - inb[None] + L, 0).astype(np.int64)
    return 2 * c_out * int(per_site.sum()), dense, run.any(axis=0)


def inc_conv2d(values, flags, th, tw, weight, stride=1, pad=0):
    """increment_ops.py:126-194 -- returns (y, y_flags, performed, dense_equiv).

    Values: the bias-free convolution of the increment (the reference sums
    only live channels per site; dead taps read exact zeros, so this is the
    same sum up to reassociation).  Masks and the meter are exact.
    """
    weight = np.asarray(weight, dtype=F32)
    c_out, c_in, kh, kw = weight.shape
    c, h, w = values.shape
    if c != c_in:
        raise ValueError(f"increment has {c} channels but conv expects {c_in}")
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    performed, dense, act = conv_meter(flags, th, tw, h, w, c_out, kh, kw, stride, pad)
    out_grid = tile_grid((c_out, ho, wo), th, tw)
    if not flags.any():
        return np.zeros((c_out, ho, wo), F32), np.zeros(out_grid, bool), 0, dense
    if flags.all():
        return dense_conv2d(values, weight, None, stride, pad), np.ones(out_grid, bool), dense, dense
    y = dense_conv2d(values, weight, None, stride, pad)
    y[:, ~act] = 0.0
    oflags = np.broadcast_to(tiles_any(act[None], th, tw), out_grid).copy()
    return y, oflags, performed, dense


def inc_conv2d_refalg(values, flags, th, tw, weight, stride=1, pad=0):
    """The reference's per-input-channel gather + sgemm loop
    (increment_ops.py:156-194), restated.  Slow by design: it is what the
    CPU baseline times."""
    weight = np.asarray(weight, dtype=F32)
    c_out, c_in, kh, kw = weight.shape
    c, h, w = values.shape
    ho, wo = conv_out_hw(h, w, kh, kw, stride, pad)
    kk = kh * kw
    dense = 2 * kk * c_in * c_out * ho * wo
    out_grid = tile_grid((c_out, ho, wo), th, tw)
    if not flags.any():
        return np.zeros((c_out, ho, wo), F32), np.zeros(out_grid, bool), 0, dense
    if flags.all():
        return dense_conv2d(values, weight, None, stride, pad), np.ones(out_grid, bool), dense, dense
    live = flags_to_pixels(flags, th, tw, h, w)
    pads = ((0, 0), (pad, pad), (pad, pad))
    livep, deadp, xp = np.pad(live, pads), np.pad(~live, pads), np.pad(values, pads)
    wmat = weight.reshape(c_out, c_in, kk)
    y = np.zeros((c_out, ho, wo), F32)
    act = np.zeros((ho, wo), bool)
    macs = 0
    taps = [(r, s) for r in range(kh) for s in range(kw)]
    for ch in np.flatnonzero(flags.reshape(c_in, -1).any(axis=1)):
        n_live = sum(livep[ch, r : r + stride * ho : stride, s : s + stride * wo : stride].astype(np.int64) for r, s in taps)
        n_dead = sum(deadp[ch, r : r + stride * ho : stride, s : s + stride * wo : stride].astype(np.int64) for r, s in taps)
        run = n_live > 0
        k_runs = int(run.sum())
        if not k_runs:
            continue
        macs += k_runs * kk - int(n_dead[run].sum())
        act |= run
        uu, vv = np.nonzero(run)
        cols = np.stack([xp[ch, uu * stride + r, vv * stride + s] for r, s in taps])
        y[:, uu, vv] += wmat[:, ch, :] @ cols
    oflags = np.broadcast_to(tiles_any(act[None], th, tw), out_grid).copy()
    return y, oflags, 2 * c_out * macs, dense


def flatten_runs(values, th, tw):
    """increment_ops.py:197-202 flatten_increment: ravel to (1,1,L) with
    runs of th*tw elements as tiles; returns the run flags."""
    run = th * tw
    flat = np.asarray(values, dtype=F32).reshape(-1)
    n = flat.size
    nr = (n + run - 1) // run
    pad = np.zeros(nr * run, bool)
    pad[:n] = flat != 0
    return pad.reshape(nr, run).any(axis=1)


def inc_linear(values, th, tw, matrix):
    """increment_ops.py:205-223 (after flatten_increment) --
    returns (y (F,), performed, dense_equiv); the output mask is all-true."""
    matrix = np.asarray(matrix, dtype=F32)
    flat = np.asarray(values, dtype=F32).reshape(-1)
    rows, cols = matrix.shape
    if cols != flat.size:
        raise ValueError(f"matrix {matrix.shape} does not apply to increment of length {flat.size}")
    run = th * tw
    live = np.repeat(flatten_runs(values, th, tw), run)[: flat.size]
    idx = np.flatnonzero(live)
    y = np.zeros(rows, F32)
    performed = 0
    if idx.size:
        y = matrix[:, idx] @ flat[idx]
        performed = 2 * rows * idx.size
    return y.astype(F32), performed, 2 * rows * cols


def inc_add(a, fa, b, fb):
    """increment_ops.py:226-229."""
    return a + b, fa | fb


def inc_activation(values, flags, acc, kind, alpha=0.01):
    """increment_ops.py:232-238 -- returns (y, flags, new_acc)."""
    fn = activation(kind, alpha)
    y = (fn(acc + values) - fn(acc)).astype(F32)
    return y, flags.copy(), acc + values


def inc_mul(a, fa, b, fb, acc_a, acc_b):
    """increment_ops.py:241-254 -- (acc_a + a) * b + acc_b * a."""
    y = (acc_a + a) * b + acc_b * a
    return y, fa | fb, acc_a + a, acc_b + b


def inc_concat(parts):
    """increment_ops.py:257-268 -- parts: list of (values, flags)."""
    return (np.concatenate([p[0] for p in parts], axis=0),
            np.concatenate([p[1] for p in parts], axis=0))


def inc_upsample(values, flags, th, tw, factor, mode="nearest"):
    """increment_ops.py:271-285 -- linear upsample of dx, mask from pixel support."""
    y = dense_upsample(values, factor, mode)
    _, h, w = values.shape
    live = flags_to_pixels(flags, th, tw, h, w)
    if mode == "nearest":
        ri = np.arange(h * factor) // factor
        ci = np.arange(w * factor) // factor
        out_live = live[:, ri][:, :, ci]
    else:
        r0, r1, _ = bilinear_taps(h, factor)
        c0, c1, _ = bilinear_taps(w, factor)
        rl = live[:, r0] | live[:, r1]
        out_live = rl[:, :, c0] | rl[:, :, c1]
    return y, tiles_any(out_live, th, tw)


def inc_maxpool(values, flags, th, tw, acc, window=(2, 2), stride=2):
    """increment_ops.py:288-310 -- returns (y, flags, new_acc)."""
    before = dense_maxpool(acc, window, stride)
    new_acc = acc + values
    y = dense_maxpool(new_acc, window, stride) - before
    c, h, w = values.shape
    wh, ww = window
    ho, wo = (h - wh) // stride + 1, (w - ww) // stride + 1
    live = flags_to_pixels(flags, th, tw, h, w)
    pooled = np.zeros((c, ho, wo), bool)
    for r in range(wh):
        for s in range(ww):
            pooled |= live[:, r : r + stride * ho : stride, s : s + stride * wo : stride]
    return y, tiles_any(pooled, th, tw), new_acc


# ---------------------------------------------------------------------------
# sparsification  (sparsify.py)
# ---------------------------------------------------------------------------


def sparsify_state(shape, tp=0.0, ema_decay=0.9, k=0.0):
    """sparsify.py:25-41 SparsifyState.__init__."""
    if tp < 0:
        raise ValueError("threshold parameter must be >= 0")
    if not (0.0 < ema_decay < 1.0):
        raise ValueError("ema_decay must lie in (0, 1)")
    return {"delta": np.zeros(shape, F32), "norm_ema": 0.0, "k": float(k),
            "tp": float(tp), "ema_decay": float(ema_decay)}


def sparsify_reset(st, dense_input):
    """sparsify.py:43-51."""
    x = np.asarray(dense_input, dtype=F32)
    st["delta"] = np.zeros(x.shape, F32)
    st["norm_ema"] = float(np.linalg.norm(x))
    if st["tp"] > 0:
        st["k"] = st["tp"] * st["norm_ema"]


def sparsify_step(values, th, tw, st):
    """sparsify.py:54-78 -- round to multiples of k with error feedback.
    Mutates ``st``; returns (y, flags)."""
    corrected = st["delta"] + values
    k = st["k"]
    if k > 0:
        k32 = F32(k)
        y = k32 * np.floor(F32(0.5) + corrected / k32)
        st["delta"] = corrected - y
    else:
        y = corrected
        st["delta"] = np.zeros(values.shape, F32)
    d = st["ema_decay"]
    st["norm_ema"] = d * st["norm_ema"] + (1.0 - d) * float(np.linalg.norm(corrected))
    if st["tp"] > 0:
        st["k"] = st["tp"] * st["norm_ema"]
    y = y.astype(F32, copy=False)
    return y, tile_flags(y, th, tw)


# ---------------------------------------------------------------------------
# events  (events.py)
# ---------------------------------------------------------------------------


def slice_window(t, tau, delta):
    """events.py:240-248 -- (tau - delta, tau] by binary search."""
    if delta <= 0:
        raise ValueError("window length must be positive")
    lo = 0 if tau - delta < 0 else int(np.searchsorted(t, tau - delta, side="right"))
    hi = int(np.searchsorted(t, tau, side="right"))
    return lo, hi


def encode(t, x, y, p, lo, hi, tau, delta, h, w, kind, bins=1):
    """events.py:251-292 -- count / timestamp / voxel encodings (float32)."""
    xs = np.asarray(x[lo:hi], np.int64)
    ys = np.asarray(y[lo:hi], np.int64)
    ps = np.asarray(p[lo:hi]).astype(F32)
    rel = (np.asarray(t[lo:hi]).astype(np.float64) - float(tau - delta)) / float(delta)
    pos = ps > 0
    if kind == "count":
        out = np.zeros((2, h, w), F32)
        np.add.at(out[0], (ys[pos], xs[pos]), 1.0)
        np.add.at(out[1], (ys[~pos], xs[~pos]), 1.0)
        return out
    if kind == "timestamp":
        out = np.zeros((2, h, w), F32)
        tn = rel.astype(F32)
        np.maximum.at(out[0], (ys[pos], xs[pos]), tn[pos])
        np.maximum.at(out[1], (ys[~pos], xs[~pos]), tn[~pos])
        return out
    if kind != "voxel":
        raise ValueError(f"unknown encoder {kind!r}")
    out = np.zeros((bins, h, w), F32)
    if hi <= lo:
        return out
    tstar = (rel * (bins - 1)).astype(F32)
    b0 = np.floor(tstar).astype(np.int64)
    frac = tstar - b0  # float64
    for b, v in ((b0, ps * (1.0 - frac)), (b0 + 1, ps * frac)):
        ok = (b >= 0) & (b < bins)
        np.add.at(out, (b[ok], ys[ok], xs[ok]), v[ok])
    return out


def step_increment(prev, cur, th, tw):
    """events.py:295-302 -- (cur - prev, exact tile flags)."""
    prev = np.asarray(prev, F32)
    cur = np.asarray(cur, F32)
    if prev.shape != cur.shape:
        raise ValueError(f"shape mismatch: {prev.shape} vs {cur.shape}")
    v = cur - prev
    return v, tile_flags(v, th, tw)


# ---------------------------------------------------------------------------
# graph runtime  (graph.py)
# ---------------------------------------------------------------------------

ACTS = ("relu", "sigmoid", "tanh", "leaky_relu")
KINDS = ACTS + ("conv", "linear", "add", "mul", "concat", "upsample", "maxpool", "sparsify", "delay")

# ``delay`` (recurrent-state extension, SURVEY.md 8(f) rank 3 -- not a reference kind; the reference
# has the recurrent primitives inc_mul / sigmoid / tanh, increment_ops.py:241-254, tensors.py:289-294,
# but no recurrent graph).  A delay node has no inputs; attrs ``source`` (a node id) and
# ``shape``.  Frame semantics: at frame t it outputs the source's value of frame t - 1 (zeros before the
# first frame), which closes ConvLSTM / ConvGRU loops h_t = cell(x_t, h_{t-1}) without a cycle in the
# per-frame DAG.  Incremental semantics (exact restatement of the frame semantics):
#   state  held = the delay's current output value, pend = (values, flags) of its next increment;
#   dense pass: output held; afterwards pend = step_increment(held, source)            (mutating pass)
#   incr step : output pend; held += pend (integrate); after the step pend = source's increment.


def topo_order(spec):
    """graph.py:137-185 -- Kahn's algorithm with a min-heap on node id."""
    inp = spec["input"].get("id", "input")
    nodes = {n["id"]: n for n in spec["nodes"]}
    indeg, users = {}, {}
    for n in spec["nodes"]:
        deps = [i for i in n["inputs"] if i != inp]
        indeg[n["id"]] = len(deps)
        for d in deps:
            users.setdefault(d, []).append(n["id"])
    heap = sorted(k for k, d in indeg.items() if d == 0)
    heapq.heapify(heap)
    order = []
    while heap:
        nid = heapq.heappop(heap)
        order.append(nodes[nid])
        for u in users.get(nid, ()):
            indeg[u] -= 1
            if indeg[u] == 0:
                heapq.heappush(heap, u)
    if len(order) != len(nodes):
        raise ValueError("cycle")
    return order


def node_shape(n, ins):
    """graph.py:266-305 _node_out_shape."""
    k = n["kind"]
    if k == "conv":
        c, h, w = ins[0]
        kh, kw = n.get("kernel", [3, 3])
        ho, wo = conv_out_hw(h, w, kh, kw, n.get("stride", 1), n.get("padding", 0))
        return (n["out_channels"], ho, wo)
    if k == "linear":
        return (n["out_features"], 1, 1)
    if k in ACTS or k in ("sparsify", "add", "mul"):
        return ins[0]
    if k == "concat":
        return (sum(s[0] for s in ins), *ins[0][1:])
    if k == "upsample":
        f = n.get("factor", 2)
        return (ins[0][0], ins[0][1] * f, ins[0][2] * f)
    if k == "maxpool":
        c, h, w = ins[0]
        wh, ww = n.get("window", [2, 2])
        st = n.get("stride", 2)
        return (c, (h - wh) // st + 1, (w - ww) // st + 1)
    if k == "delay":
        return tuple(int(v) for v in n["shape"])
    raise ValueError(k)


class OracleGraph:
    """graph.py:423-693 Graph session, restated over plain numpy state.

    ``spec`` is the ModelSpec YAML dict (graph.py:232-256 schema);
    ``weights`` maps ``<id>.weight`` / ``<id>.bias`` to arrays.
    ``conv_impl`` selects ``inc_conv2d`` ("fast") or the reference loop
    ("refalg").
    """

    def __init__(self, spec, weights, refresh_interval=64, conv_impl="fast"):
        self.spec = spec
        self.input_id = spec["input"].get("id", "input")
        self.input_shape = tuple(spec["input"]["shape"])
        t = spec.get("tile", [6, 6])
        self.th, self.tw = int(t[0]), int(t[1])
        self.out_ids = [spec["output"], *spec.get("aux_outputs", [])]
        self.refresh_interval = int(refresh_interval) if refresh_interval else 0
        self.order = topo_order(spec)
        self.shapes = {self.input_id: self.input_shape}
        for n in self.order:
            self.shapes[n["id"]] = node_shape(n, [self.shapes[i] for i in n["inputs"]])
        self.w = {k: np.asarray(v, F32) for k, v in weights.items()}
        self.conv = inc_conv2d if conv_impl == "fast" else inc_conv2d_refalg
        self.state = {}
        self.meter = {}
        self.ff = {}
        for n in self.order:
            nid, k = n["id"], n["kind"]
            ish = self.shapes[n["inputs"][0]] if n["inputs"] else None
            if k in ACTS or k == "maxpool":
                self.state[nid] = {"acc": np.zeros(ish, F32)}
            elif k == "mul":
                self.state[nid] = {"acc": np.zeros(ish, F32), "acc2": np.zeros(self.shapes[n["inputs"][1]], F32)}
            elif k == "sparsify":
                self.state[nid] = sparsify_state(ish, n.get("tp", 0.0), n.get("ema_decay", 0.9))
            elif k == "delay":
                sh = self.shapes[nid]
                self.state[nid] = {"held": np.zeros(sh, F32), "pv": np.zeros(sh, F32),
                                   "pf": np.zeros(tile_grid(sh, self.th, self.tw), bool)}
            if k in ("conv", "linear"):
                self.meter[nid] = [0, 0]
                self.ff[nid] = [0.0, 0.0, 0]  # last, sum, n
        self.step_count = 0
        self.refresh_due = False
        self.initialized = False
        self.baseline, self.y_run = {}, {}

    # graph.py:503-550
    def _dense(self, x, mutate):
        x = np.asarray(x, F32)
        vals = {self.input_id: x}
        for n in self.order:
            nid, k = n["id"], n["kind"]
            ins = [vals[i] for i in n["inputs"]]
            if k == "conv":
                y = dense_conv2d(ins[0], self.w[nid + ".weight"], self.w.get(nid + ".bias"),
                                 n.get("stride", 1), n.get("padding", 0))
                if mutate:
                    kh, kw = n.get("kernel", [3, 3])
                    de = 2 * kh * kw * ins[0].shape[0] * y.size
                    self.meter[nid][0] += de
                    self.meter[nid][1] += de
            elif k == "linear":
                wm = self.w[nid + ".weight"]
                y = dense_linear(ins[0].reshape(-1), wm, self.w.get(nid + ".bias")).reshape(self.shapes[nid])
                if mutate:
                    de = 2 * wm.shape[0] * wm.shape[1]
                    self.meter[nid][0] += de
                    self.meter[nid][1] += de
            elif k in ACTS:
                y = activation(k, n.get("alpha", 0.01))(ins[0])
                if mutate:
                    self.state[nid]["acc"] = ins[0].copy()
            elif k == "sparsify":
                y = ins[0]
                if mutate:
                    sparsify_reset(self.state[nid], ins[0])
            elif k == "add":
                y = ins[0] + ins[1]
            elif k == "mul":
                y = ins[0] * ins[1]
                if mutate:
                    self.state[nid]["acc"] = ins[0].copy()
                    self.state[nid]["acc2"] = ins[1].copy()
            elif k == "concat":
                y = np.concatenate(ins, axis=0)
            elif k == "upsample":
                y = dense_upsample(ins[0], n.get("factor", 2), n.get("mode", "nearest"))
            elif k == "maxpool":
                y = dense_maxpool(ins[0], tuple(n.get("window", [2, 2])), n.get("stride", 2))
                if mutate:
                    self.state[nid]["acc"] = ins[0].copy()
            elif k == "delay":
                y = self.state[nid]["held"].copy()
            else:
                raise ValueError(k)
            vals[nid] = y
        if mutate:
            for n in self.order:
                if n["kind"] == "delay":
                    st = self.state[n["id"]]
                    st["pv"], st["pf"] = step_increment(st["held"], vals[n["source"]], self.th, self.tw)
        return vals

    def dense_oracle(self, x):
        return self._dense(x, False)[self.out_ids[0]]

    def dense_pass(self, x):
        vals = self._dense(x, True)
        for o in self.out_ids:
            self.baseline[o] = vals[o].copy()
            self.y_run[o] = vals[o].copy()
        self.step_count = 0
        self.refresh_due = False
        self.initialized = True
        return vals[self.out_ids[0]]

    refresh = dense_pass

    # graph.py:573-630
    def incr_step(self, values, flags, trace=None):
        if not self.initialized:
            raise ValueError("incr_step called before any dense_pass")
        th, tw = self.th, self.tw
        vals = {self.input_id: (np.asarray(values, F32), np.asarray(flags, bool))}
        step = {}
        for n in self.order:
            nid, k = n["id"], n["kind"]
            ins = [vals[i] for i in n["inputs"]]
            st = self.state.get(nid)
            if k == "conv":
                self._observe(nid, ins[0][1])
                y, f, perf, de = self.conv(ins[0][0], ins[0][1], th, tw, self.w[nid + ".weight"],
                                           n.get("stride", 1), n.get("padding", 0))
                step[nid] = (perf, de)
                out = (y, f)
            elif k == "linear":
                self._observe(nid, ins[0][1])
                y, perf, de = inc_linear(ins[0][0], th, tw, self.w[nid + ".weight"])
                step[nid] = (perf, de)
                shp = self.shapes[nid]
                out = (y.reshape(shp), np.ones(tile_grid(shp, th, tw), bool))
            elif k in ACTS:
                y, f, st["acc"] = inc_activation(ins[0][0], ins[0][1], st["acc"], k, n.get("alpha", 0.01))
                out = (y, f)
            elif k == "sparsify":
                out = sparsify_step(ins[0][0], th, tw, st)
            elif k == "add":
                out = inc_add(ins[0][0], ins[0][1], ins[1][0], ins[1][1])
            elif k == "mul":
                y, f, st["acc"], st["acc2"] = inc_mul(ins[0][0], ins[0][1], ins[1][0], ins[1][1], st["acc"], st["acc2"])
                out = (y, f)
            elif k == "concat":
                out = inc_concat(ins)
            elif k == "upsample":
                out = inc_upsample(ins[0][0], ins[0][1], th, tw, n.get("factor", 2), n.get("mode", "nearest"))
            elif k == "maxpool":
                y, f, st["acc"] = inc_maxpool(ins[0][0], ins[0][1], th, tw, st["acc"],
                                              tuple(n.get("window", [2, 2])), n.get("stride", 2))
                out = (y, f)
            elif k == "delay":
                out = (st["pv"], st["pf"])
                st["held"] = integrate(st["held"], st["pv"], st["pf"], th, tw)
            else:
                raise ValueError(k)
            vals[nid] = out
            if trace is not None:
                trace[nid] = out
        for n in self.order:  # the next step's delayed increments
            if n["kind"] == "delay":
                sv, sf = vals[n["source"]]
                self.state[n["id"]]["pv"], self.state[n["id"]]["pf"] = sv.copy(), np.asarray(sf, bool).copy()
        for o in self.out_ids:
            self.y_run[o] = integrate(self.y_run[o], vals[o][0], vals[o][1], th, tw)
        for nid, (perf, de) in step.items():
            self.meter[nid][0] += perf
            self.meter[nid][1] += de
        self.step_count += 1
        if self.refresh_interval:
            self.refresh_due = self.step_count >= self.refresh_interval
        report = {"per_node": step, "false_tile_frac": {nid: self.ff[nid][0] for nid in self.ff}}
        return vals[self.out_ids[0]], self.y_run[self.out_ids[0]].copy(), report

    def _observe(self, nid, flags):
        """graph.py:632-636."""
        ff = false_fraction(flags)
        rec = self.ff[nid]
        rec[0] = ff
        rec[1] += ff
        rec[2] += 1

    def drift(self, oracle_y):
        """graph.py:646-654."""
        y = self.y_run[self.out_ids[0]]
        return float(np.max(np.abs(y - np.asarray(oracle_y, F32)))) if y.size else 0.0

    def flop_report(self):
        """graph.py:656-669 -- cumulative (performed, dense_equiv) per node."""
        return {nid: tuple(v) for nid, v in self.meter.items()}

    def state_fingerprint(self):
        """graph.py:678-693."""
        out = {}
        for n in self.order:
            nid = n["id"]
            st = self.state.get(nid)
            if st is None:
                continue
            if "acc" in st:
                out[nid + ".acc"] = st["acc"].copy()
            if "acc2" in st:
                out[nid + ".acc2"] = st["acc2"].copy()
            if "delta" in st:
                out[nid + ".delta"] = st["delta"].copy()
                out[nid + ".norm"] = np.asarray([st["norm_ema"], st["k"]], np.float64)
            if "held" in st:
                out[nid + ".held"] = st["held"].copy()
                out[nid + ".pend"] = st["pv"].copy()
        for o in self.out_ids:
            if o in self.y_run:
                out[o + ".y_run"] = self.y_run[o].copy()
                out[o + ".baseline"] = self.baseline[o].copy()
        return out
