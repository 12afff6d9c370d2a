"""FP16 rounding and the column range guard (oracle side).

* fl16: IEEE binary16 round-to-nearest-even (§2.1: "we use FP16 format
  supported by NVIDIA TensorCore"). numpy's float16 conversion is a library primitive used
  as one step; tests pin it to SPEC.md:47-50 examples and the IEEE closed form.
* pow2_colscale: per-column power-of-two scale s_j = 2^(-floor(log2 max_i |X_ij|)), DESIGN.md
  reading R-A4 (paper silent on FP16 range). With it every scaled column has max in [1, 2).
"""
from __future__ import annotations

import numpy as np


def fl16(x: np.ndarray) -> np.ndarray:
    """Round to IEEE binary16 (RNE, subnormals kept, overflow to inf), returned as float64."""
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def pow2_colscale(x: np.ndarray) -> np.ndarray:
    """s_j = 2^(-floor(log2(max_i |x_ij|))); s_j = 1 for an all-zero column (R-A4)."""
    mx = np.max(np.abs(x), axis=0)
    s = np.ones(x.shape[1])
    nz = mx > 0
    # frexp: mx = f * 2^e with f in [0.5, 1)  =>  floor(log2 mx) = e - 1, exactly.
    _, e = np.frexp(mx[nz])
    s[nz] = np.ldexp(1.0, -(e - 1))
    return s
