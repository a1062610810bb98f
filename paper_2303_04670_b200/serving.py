"""Host-I/O-overlapped serving loop over a :class:`~paper_2303_04670_b200.graph.Graph`.

The reference's timed loop (reference bench.py:196-209) is strictly serial: encode the
next window, ``step_increment``, ``incr_step``, read the output.  On a GPU the host
copies of one step can run under the compute of its neighbours: while step i runs on
the compute stream, a copy stream uploads frame i + 1 and downloads step i - 1's
integrated output.  Every step still moves its own input host -> device and its own
result device -> host; only the ordering changes, so each step's output is bit-identical
to the serial loop (tests/test_gpu_serving.py).

Buffers: a ring of three device frames (frame i is ``cur`` of step i and ``prev`` of
step i + 1, so the upload of frame i + 2 may only overwrite frame i - 1 after step i
finished), and two device snapshots of the integrated output (the graph updates it in
place every step).
"""

from __future__ import annotations

import numpy as np
import torch


class StreamPipeline:
    """Run consecutive increments of a graph with uploads / downloads overlapped.

    ``host_frames``: pinned host tensor ``(n + 1, S, C, H, W)`` (``(n + 1, C, H, W)`` for
    one session) of encoded windows; frame 0 is the dense-pass input.
    ``out_host``: pinned host tensor ``(n, *integrated_output_shape)``; row i - 1 receives
    the integrated output after increment i.
    A refresh (dense pass) runs in-line whenever the graph reports it due, as in the
    reference's bench loop.
    """

    def __init__(self, graph):
        self.g = graph
        dev = graph.device
        self.copy = torch.cuda.Stream(device=dev)
        self.compute = torch.cuda.current_stream(dev)

    def run(self, host_frames: torch.Tensor, out_host: torch.Tensor, *, dense_first: bool = True) -> int:
        g = self.g
        n = host_frames.shape[0] - 1
        if n < 1:
            return 0
        if not (host_frames.is_pinned() and out_host.is_pinned()):
            raise ValueError("StreamPipeline: host_frames and out_host must be pinned")
        y = g._y_run[g.output_ids[0]]
        one = g.S == 1 and host_frames.dim() == 4
        frames = [torch.empty(host_frames.shape[1:], dtype=host_frames.dtype, device=g.device) for _ in range(3)]
        snaps = [torch.empty_like(y) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(3)]     # frame k uploaded
        ev_done = [torch.cuda.Event() for _ in range(3)]   # step using frame k as `cur` finished
        ev_snap = [torch.cuda.Event() for _ in range(2)]   # snapshot k written
        ev_out = [torch.cuda.Event() for _ in range(2)]    # snapshot k downloaded
        cs, cp = self.compute, self.copy

        def upload(i):
            k = i % 3
            with torch.cuda.stream(cp):
                if i >= 3:
                    cp.wait_event(ev_done[(i - 2) % 3])  # frame i - 3 was `prev` of step i - 2
                frames[k].copy_(host_frames[i], non_blocking=True)
                ev_in[k].record(cp)

        upload(0)
        if n >= 1:
            upload(1)
        cs.wait_event(ev_in[0])
        if dense_first:
            g.dense_pass(frames[0])
        ev_done[0].record(cs)
        for i in range(1, n + 1):
            if i + 1 <= n:
                upload(i + 1)
            k, kp = i % 3, (i - 1) % 3
            cs.wait_event(ev_in[k])
            g.step_from_encodings(frames[kp], frames[k])
            if g.refresh_due:
                g.dense_pass(frames[k])
            j = i % 2
            if i >= 3:
                cs.wait_event(ev_out[j])  # snapshot j's previous download finished
            snaps[j].copy_(y)
            ev_snap[j].record(cs)
            ev_done[k].record(cs)
            with torch.cuda.stream(cp):
                cp.wait_event(ev_snap[j])
                out_host[i - 1].copy_(snaps[j][0] if one else snaps[j], non_blocking=True)
                ev_out[j].record(cp)
            if i >= 2:
                ev_out[(i - 1) % 2].synchronize()  # the host holds step i - 1's result
        ev_out[n % 2].synchronize()
        return n


def window_bounds(t, taus, delta):
    """(lo, hi) event-index arrays of every window (tau - delta, tau] of the time-sorted timestamps t
    (slice_window, events.py:240-248, for all taus at once): one vectorised searchsorted per edge, the keys in
    t's own dtype (a Python-int key makes numpy convert the whole array on every call)."""
    t = np.asarray(t)
    ends = np.asarray(taus, dtype=np.int64)
    starts = ends - int(delta)
    lo = np.searchsorted(t, np.maximum(starts, 0).astype(t.dtype), side="right")
    return np.where(starts < 0, 0, lo), np.searchsorted(t, ends.astype(t.dtype), side="right")


class EventPipeline:
    """Serving loop from raw events: per step, only the newly arrived
    packed EVB records of every session cross PCIe.

    The reference path re-reads and re-encodes every window on the host (read_events,
    events.py:185-206; encode, events.py:251-292) and ships dense tensors.  Here each session
    keeps its recent events in a device ring (``ring`` slots per column, a power of two); every
    step the host appends the records that arrived since the last window end -- 13 bytes per
    event, ``{u64 t, u16 x, u16 y, i8 p}`` (events.py:35-37) -- to a pinned staging block with
    a small per-session descriptor, one H2D copy moves the block, and on an ingest stream
    ``evc_ingest_ring`` unpacks it into the rings and ``evc_encode_windows`` bins every session's
    window (count + timestamp, bit-identical to ``encode``) into one of three encoding buffers --
    one step ahead, overlapping the previous step's compute --; on the compute stream
    ``step_from_encodings`` forms the increment and runs the step (a dense pass for the
    first window and whenever a refresh is due).  The integrated output of every step is read
    back as in :class:`StreamPipeline`.  Uploads of step i + 1 overlap step i's compute.
    """

    MODES = {"count": 1, "timestamp": 2, "count+timestamp": 3}

    def __init__(self, graph, sensor_size, mode: str = "count+timestamp", window_us: int = 50_000,
                 ring: int = 1 << 17, max_new: int | None = None):
        from . import _lib

        if mode not in self.MODES:
            raise ValueError(f"unknown ingest mode {mode!r} (count, timestamp, count+timestamp)")
        g = self.g = graph
        self.mode = self.MODES[mode]
        c = 4 if self.mode == 3 else 2
        self.H, self.W = (int(v) for v in sensor_size)
        if tuple(g.input_shape) != (c, self.H, self.W):
            raise ValueError(f"graph input {g.input_shape} does not match {mode} encodings of {self.H}x{self.W}")
        if ring & (ring - 1):
            raise ValueError("ring must be a power of two")
        self.window_us, self.ring = int(window_us), int(ring)
        self.max_new = int(max_new) if max_new else self.ring  # (the first window arrives whole)
        S, dev = g.S, g.device
        self.cols = (torch.zeros(S * ring, dtype=torch.int64, device=dev), torch.zeros(S * ring, dtype=torch.int16, device=dev),
                     torch.zeros(S * ring, dtype=torch.int16, device=dev), torch.zeros(S * ring, dtype=torch.int8, device=dev))
        self.enc = [torch.zeros((S, c, self.H, self.W), dtype=torch.float32, device=dev) for _ in range(3)]
        self.meta = 7 * S  # int64 words: desc (3 per session) + windows (4 per session)
        nbytes = 8 * self.meta + S * self.max_new * 13
        self.host = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(2)]
        self.dev_stage = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
        self.copy = torch.cuda.Stream(device=dev)
        self.ingest = torch.cuda.Stream(device=dev)
        self.compute = torch.cuda.current_stream(dev)
        self.lib = _lib.lib()
        self.h2d_bytes = []

    def _fill(self, k, recs, bounds, prev_hi, tau):
        """Stage step data into host buffer k: per-session new records + desc + windows."""
        S = self.g.S
        buf = self.host[k].numpy()
        meta = buf[: 8 * self.meta].view(np.int64)
        off = 8 * self.meta
        first, most = 0, 0
        for s in range(S):
            lo, hi = bounds[s]
            a = prev_hi[s] if prev_hi is not None else lo
            n = hi - a
            if n > self.max_new:
                raise ValueError(f"session {s}: {n} new events exceed max_new={self.max_new}")
            if hi - min(lo, a) > self.ring:
                raise ValueError(f"session {s}: window of {hi - lo} events exceeds the ring ({self.ring})")
            raw = recs[s][a:hi].view(np.uint8).reshape(-1)
            buf[off + 13 * first: off + 13 * (first + n)] = raw
            meta[3 * s: 3 * s + 3] = (first, n, a)
            meta[3 * S + 4 * s: 3 * S + 4 * s + 4] = (lo, hi, tau[s], self.window_us)
            first += n
            most = max(most, n)
        return 8 * self.meta + 13 * first, most

    def run(self, records, t_host, taus, out_host: torch.Tensor) -> int:
        """records[s]: the session's packed EVB records (numpy, _EVB_RECORD dtype, time-sorted);
        t_host[s]: their timestamps; taus[s]: window ends tau_0 .. tau_n.  Step 0 is the dense pass
        on window 0; out_host (pinned, (n, *output)) row i - 1 receives the integrated output after
        increment i.  Returns n."""
        from . import _lib

        g, S = self.g, self.g.S
        n = len(taus[0]) - 1
        if not out_host.is_pinned():
            raise ValueError("EventPipeline: out_host must be pinned")
        y = g._y_run[g.output_ids[0]]
        one = S == 1 and out_host.dim() == y.dim()
        snaps = [torch.empty_like(y) for _ in range(2)]
        ev_h2d = [torch.cuda.Event() for _ in range(2)]
        ev_used = [torch.cuda.Event() for _ in range(2)]
        ev_snap = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        cs, cp = self.compute, self.copy
        t, x, yy, p = self.cols
        c, H, W = g.input_shape
        stride = c * H * W
        prev_hi = None
        self.h2d_bytes = []

        lo_all, hi_all = zip(*(window_bounds(t_host[s], taus[s], self.window_us) for s in range(S)))

        def bounds_of(i):
            return [(int(lo_all[s][i]), int(hi_all[s][i])) for s in range(S)]

        def stage(i, bnds, prev):
            k = i % 2
            if i >= 2:
                ev_h2d[k].synchronize()  # host buffer k's previous upload has left
            nb, nev = self._fill(k, records, bnds, prev, [taus[s][i] for s in range(S)])  # nev: most per session
            with torch.cuda.stream(cp):
                if i >= 2:
                    cp.wait_event(ev_used[k])  # device buffer k's previous contents were consumed
                self.dev_stage[k][:nb].copy_(self.host[k][:nb], non_blocking=True)
                ev_h2d[k].record(cp)
            self.h2d_bytes.append(nb)
            return nev

        # ingest + binning run on their own stream, one step ahead: the window of step i + 1 is binned
        # while step i computes.  Encodings rotate through three buffers: step j reads windows j - 1 and j,
        # so window i's buffer (= window i - 3's) was last read by step i - 2.
        ing = self.ingest
        ev_enc = [torch.cuda.Event() for _ in range(2)]
        ev_step = [torch.cuda.Event() for _ in range(2)]

        def ingest(i, bnds, pend):
            k = i % 2
            with torch.cuda.stream(ing):
                ing.wait_event(ev_h2d[k])
                if i >= 2:
                    ing.wait_event(ev_step[(i - 2) % 2])  # buffer i % 3 was last read by step i - 2
                st = self.dev_stage[k]
                meta = st.data_ptr()
                _lib.check(self.lib.evc_ingest_ring(meta + 8 * self.meta, meta, max(pend, 1), self.ring, t.data_ptr(),
                                                    x.data_ptr(), yy.data_ptr(), p.data_ptr(), S, _lib.stream_ptr()),
                           "ingest_ring")
                wmax = max(b[1] - b[0] for b in bnds)
                _lib.check(self.lib.evc_encode_windows(t.data_ptr(), x.data_ptr(), yy.data_ptr(), p.data_ptr(), self.ring,
                                                       meta + 8 * 3 * S, max(wmax, 1), H, W, self.mode,
                                                       self.enc[i % 3].data_ptr(), stride, S, _lib.stream_ptr()),
                           "encode_windows")
                ev_used[k].record(ing)
                ev_enc[k].record(ing)

        bnds = bounds_of(0)
        ingest(0, bnds, stage(0, bnds, None))
        for i in range(n + 1):
            if i + 1 <= n:  # stage the next step's records (host fill + H2D on the copy stream)
                b1 = bounds_of(i + 1)
                pend = stage(i + 1, b1, [b[1] for b in bnds])
                bnds = b1
            cs.wait_event(ev_enc[i % 2])
            cur, prv = self.enc[i % 3], self.enc[(i - 1) % 3]
            if i == 0:
                g.dense_pass(cur if S > 1 else cur[0])
            else:
                g.step_from_encodings(prv if S > 1 else prv[0], cur if S > 1 else cur[0])
                if g.refresh_due:
                    g.dense_pass(cur if S > 1 else cur[0])
            ev_step[i % 2].record(cs)
            if i + 1 <= n:  # bin window i + 1 while step i computes
                ingest(i + 1, bnds, pend)
            if i == 0:
                continue
            j = i % 2
            if i >= 3:
                cs.wait_event(ev_out[j])
            snaps[j].copy_(y)
            ev_snap[j].record(cs)
            with torch.cuda.stream(cp):
                cp.wait_event(ev_snap[j])
                out_host[i - 1].copy_(snaps[j][0] if one else snaps[j], non_blocking=True)
                ev_out[j].record(cp)
            if i >= 2:
                ev_out[(i - 1) % 2].synchronize()
        ev_out[n % 2].synchronize()
        return n
