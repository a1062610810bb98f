"""evc_fill_segments (the dense refresh's batched resets, graph.py:503-565 semantics): every byte of every
segment takes the segment's value, nothing outside a segment changes -- unaligned heads and tails, empty,
one-byte and multi-MB segments, several CTAs per segment and fewer CTAs than segments."""

import numpy as np
import pytest
import torch

from paper_2303_04670_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_blocks", [1, 7, 592])
def test_fill_segments_edges(n_blocks):
    lib = _lib.lib()
    rng = np.random.default_rng(n_blocks)
    host = rng.integers(0, 256, size=5_000_000, dtype=np.uint8)
    buf = torch.from_numpy(host.copy()).cuda()
    base = buf.data_ptr()
    # (offset, bytes, value): misaligned starts / ends, a 1-byte and an empty segment, a large one
    segs = [(3, 29, 0), (64, 16, 1), (97, 1, 255), (200, 0, 7), (1001, 4_000_000, 0), (4_000_123, 17, 0xAB),
            (4_999_990, 10, 3)]
    tab = torch.tensor([(base + o, n, v) for o, n, v in segs], dtype=torch.int64).cuda()
    _lib.check(lib.evc_fill_segments(tab.data_ptr(), len(segs), n_blocks, _lib.stream_ptr()), "fill_segments")
    got = buf.cpu().numpy()
    want = host.copy()
    for o, n, v in segs:
        want[o:o + n] = v & 0xFF
    assert np.array_equal(got, want)
