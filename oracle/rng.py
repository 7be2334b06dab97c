"""Counter-based Gaussian test matrix Omega_k — ORACLE side (test infrastructure only).

Alg. 1 line 1 draws a fresh Gaussian Omega each call; SURVEY A6 fixes a
seed schedule (seed, stream) so the oracle and the GPU draw the same Omega without
sharing code: this file and csrc/ each implement the same published generator.

Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3"):
  round:  (hi0,lo0) = mulhilo(0xD2511F53, c0); (hi1,lo1) = mulhilo(0xCD9E8D57, c2)
          c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
  key bump between rounds: k0 += 0x9E3779B9, k1 += 0xBB67AE85 (10 rounds, 9 bumps).
Entry Omega[i, j] (m x l, column-major linear index L = j*m + i) uses the pair p = L >> 1:
  counter = (p lo32, p hi32, stream lo32, stream hi32), key = (seed lo32, seed hi32)
  a = ((x0 << 32) | x1) >> 11, b = ((x2 << 32) | x3) >> 11      (53-bit integers)
  u1 = (a + 0.5) 2^-53 in (0,1],  u2 = b 2^-53 in [0,1)
  Box-Muller: r = sqrt(-2 ln u1); even L -> r cos(2 pi u2), odd L -> r sin(2 pi u2).
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit values."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & _MASK for v in (c0, c1, c2, c3))
    k0 &= 0xFFFFFFFF
    k1 &= 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0)
    return c0, c1, c2, c3


def gaussian_omega(m: int, ell: int, seed: int, stream: int) -> np.ndarray:
    """Omega (m x ell, column-major fp64) for (seed, stream)."""
    L = np.arange(m * ell, dtype=np.uint64)
    p = L >> np.uint64(1)
    x0, x1, x2, x3 = philox4x32_10(p & _MASK, p >> np.uint64(32),
                                   np.full_like(p, stream & 0xFFFFFFFF),
                                   np.full_like(p, (stream >> 32) & 0xFFFFFFFF),
                                   seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    a = ((x0 << np.uint64(32)) | x1) >> np.uint64(11)
    b = ((x2 << np.uint64(32)) | x3) >> np.uint64(11)
    u1 = (a.astype(np.float64) + 0.5) * 2.0 ** -53
    u2 = b.astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * np.pi * u2
    z = np.where((L & np.uint64(1)) == 0, r * np.cos(th), r * np.sin(th))
    return np.asfortranarray(z.reshape(ell, m).T)


# Omega stream schedule: stream 0 = initial point, stream k+1 = outer iteration k.
def omega_stream(k: int) -> int:
    return 0 if k < 0 else k + 1
