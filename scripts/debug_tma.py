"""Bring-up bisection of the TMA region conv kernel: one subprocess per debug flag set."""

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2303_04670_b200 as evc
from paper_2303_04670_b200 import _lib
from oracle import evincr_np as O
lib = _lib.lib()
lib.evc_debug_flags.argtypes = [_lib.C.c_int32]
lib.evc_debug_flags(%d)
rng = np.random.default_rng(0)
x = rng.standard_normal((8, 16, 32)).astype(np.float32)
w = rng.standard_normal((16, 8, 3, 3)).astype(np.float32)
y = evc.dense_conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), None, 1, 1)
torch.cuda.synchronize()
ref = O.dense_conv2d(x, w, None, 1, 1)
print("RESULT max err", float(np.abs(y.cpu().numpy() - ref).max()), "max ref", float(np.abs(ref).max()))
"""


def main():
    for flags in [int(a) for a in sys.argv[1:]] or [0, 1, 2, 4, 6, 7, 8, 9]:
        p = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), flags)], capture_output=True, text=True,
                           timeout=120)
        tail = (p.stdout + p.stderr).strip().splitlines()
        msg = [ln for ln in tail if "RESULT" in ln or "Error" in ln or "error" in ln][-1:] or tail[-1:]
        print(f"flags={flags}: rc={p.returncode} {msg}", flush=True)


if __name__ == "__main__":
    main()
