"""Shared helpers for the test-suite (golden fixture access, tolerances)."""

from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def unpack(npz, prefix):
    """Inverse of make_golden.pack for one prefix: returns a nested dict."""
    out = {}
    pre = prefix + "/"
    for k in npz.files:
        if not k.startswith(pre):
            continue
        parts = k[len(pre):].split("/")
        d = out
        for p in parts[:-1]:
            d = d.setdefault(p, {})
        d[parts[-1]] = npz[k]
    return out



def close(a, b, tol=1e-5):
    """Normwise check: max|a-b| <= tol * max(1, max|b|)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    return float(np.abs(a - b).max() if a.size else 0.0) <= tol * scale


def max_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    return float(np.abs(a - b).max() if a.size else 0.0) / scale
