"""BASELINE.json configs[4] (large dense QP, column-sharded) — shardable, device-resident input
generator.  Input generation only: none of the method's arithmetic lives here.

Recipe (BASELINE configs[4]):
    A = W H + s G,   W (m x r), H (r x n_gen), G (m x n_gen) iid N(0,1),  r = 100, s = 1e-2
    q ~ U[0,1] with exactly floor(0.3 n_gen) zeros (seeded permutation),
    x0 ~ U[0.5,1.5]^n_gen, y0 ~ N(0,1)^m, z0 ~ U[0.5,1.5]^n_gen,
    b = A x0,  c = A^T y0 + z0 - q o x0          (feasible primal-dual point, as config 0).
The QP uses the columns [0, n) of the generator (n = n_gen: the full config; n = 50000: the
one-GPU slice of A25, a self-consistent QP with the same y0 and restricted x0, z0, q).

A at full size is 160 GB, so it is never drawn by a sequential generator: every entry of W, H
and G is a counter-based Philox4x32-10 draw keyed by (seed, matrix id) with the entry's global
column-major index as the counter, so any rank generates its own column shard
independently, on the device, and the instance does not depend on the number of ranks.  The
small n-/m-vectors come from numpy default_rng(seed) in the fixed order q, zero-permutation,
x0, y0, z0 (drawn at n_gen, then restricted).

Philox4x32-10 (Salmon et al., SC'11) is re-implemented here on torch int64 tensors (32-bit
values, mulhilo by 16-bit limbs so that no product exceeds 2^49), independently of oracle/rng.py
and of csrc/.  Normal pair p (entries 2p, 2p+1): counter (p lo, p hi, id, 0), key (seed, 0);
u1 = (a + 0.5) 2^-53, u2 = b 2^-53 from the 53-bit integers a = (x0 x1) >> 11, b = (x2 x3) >> 11;
Box-Muller r = sqrt(-2 ln u1): even entry r cos(2 pi u2), odd entry r sin(2 pi u2).
The integer part is bit-identical on CPU and GPU; log/cos/sin may differ in the last ulp between
the two, so a host regeneration of a device shard agrees to ~1e-16 relative.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

W_ID, H_ID, G_ID = 1, 2, 3
RANK, NOISE = 100, 1e-2
FULL_M, FULL_N, SLICE_N, ELL = 50000, 400000, 50000, 200

_M0, _M1 = 0xD2511F53, 0xCD9E8D57
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK32 = 0xFFFFFFFF


def _mulhilo(a: torch.Tensor, mult: int):
    """(hi, lo) 32-bit halves of a * mult for int64 tensors holding values < 2^32."""
    a_lo = a & 0xFFFF
    a_hi = a >> 16
    p1 = a_lo * mult                      # < 2^48
    t = a_hi * mult + (p1 >> 16)          # < 2^49
    hi = t >> 16
    lo = ((t & 0xFFFF) << 16) | (p1 & 0xFFFF)
    return hi, lo


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 on int64 tensors holding 32-bit values (10 rounds, 9 key bumps)."""
    k0 &= _MASK32
    k1 &= _MASK32
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & _MASK32
            k1 = (k1 + _W1) & _MASK32
        hi0, lo0 = _mulhilo(c0, _M0)
        hi1, lo1 = _mulhilo(c2, _M1)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def normals(seed: int, mid: int, start: int, count: int, device="cpu") -> torch.Tensor:
    """Entries [start, start + count) of the N(0,1) stream (seed, matrix id), fp64."""
    if count <= 0:
        return torch.empty(0, dtype=torch.float64, device=device)
    p0 = start // 2
    p1 = (start + count + 1) // 2
    p = torch.arange(p0, p1, dtype=torch.int64, device=device)
    zero = torch.zeros_like(p)
    x0, x1, x2, x3 = philox4x32_10(p & _MASK32, p >> 32, zero + mid, zero, seed, 0)
    a = ((x0 << 21) | (x1 >> 11)).to(torch.float64)   # top 53 bits of (x0 x1)
    b = ((x2 << 21) | (x3 >> 11)).to(torch.float64)
    del x0, x1, x2, x3, p, zero
    u1 = (a + 0.5) * 2.0 ** -53
    u2 = b * 2.0 ** -53
    r = torch.sqrt(-2.0 * torch.log(u1))
    th = (2.0 * math.pi) * u2
    z = torch.stack((r * torch.cos(th), r * torch.sin(th)), dim=1).reshape(-1)
    off = start - 2 * p0
    return z[off:off + count]


def vectors(m: int, n_gen: int, seed: int = 4):
    """q, x0, z0 (n_gen) and y0 (m) from numpy default_rng(seed), fixed draw order."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(0.0, 1.0, n_gen)
    q[rng.permutation(n_gen)[: int(0.3 * n_gen)]] = 0.0      # floor(0.3 n) zeros (A22)
    x0 = rng.uniform(0.5, 1.5, n_gen)
    y0 = rng.standard_normal(m)
    z0 = rng.uniform(0.5, 1.5, n_gen)
    return q, x0, y0, z0


@dataclass
class Shard:
    """Columns [lo, hi) of a config-4 instance in the library layout.

    At : (hi - lo, lda) fp64 tensor == A[:, lo:hi] column-major with leading dimension lda
    b_part : A[:, lo:hi] x0[lo:hi] (m) — sum over ranks gives b
    q, c, x0, z0 : this shard's slices (tensors on the same device); y0 : m
    """
    m: int
    n: int
    lo: int
    hi: int
    lda: int
    At: torch.Tensor
    b_part: torch.Tensor
    q: torch.Tensor
    c: torch.Tensor
    x0: torch.Tensor
    y0: torch.Tensor
    z0: torch.Tensor


def generate_shard(m: int, n: int, lo: int, hi: int, n_gen: Optional[int] = None, seed: int = 4,
                   device="cpu", lda_multiple: int = 32, chunk_elems: int = 1 << 25,
                   rank_r: int = RANK, noise: float = NOISE) -> Shard:
    """Generate columns [lo, hi) of the QP on columns [0, n) of the config-4 generator."""
    n_gen = n if n_gen is None else n_gen
    assert 0 <= lo <= hi <= n <= n_gen
    r = min(rank_r, m, n_gen)
    qn, x0n, y0n, z0n = vectors(m, n_gen, seed)
    lda = ((m + lda_multiple - 1) // lda_multiple) * lda_multiple
    ncol = hi - lo
    At = torch.zeros((max(ncol, 1), lda), dtype=torch.float64, device=device)[:ncol] if ncol else \
        torch.zeros((0, lda), dtype=torch.float64, device=device)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    # W^T (r x m): W[i, k] is entry i + m k of stream W_ID
    Wt = normals(seed, W_ID, 0, m * r, device).reshape(r, m)
    q, x0, z0, y0 = dev(qn[lo:hi]), dev(x0n[lo:hi]), dev(z0n[lo:hi]), dev(y0n)
    b_part = torch.zeros(m, dtype=torch.float64, device=device)
    c = torch.empty(ncol, dtype=torch.float64, device=device)
    step = max(1, chunk_elems // max(m, 1))
    for j0 in range(lo, hi, step):
        j1 = min(hi, j0 + step)
        k = j1 - j0
        Ht = normals(seed, H_ID, r * j0, r * k, device).reshape(k, r)          # H[:, j0:j1]^T
        blk = Ht @ Wt                                                          # (W H)[:, j0:j1]^T
        blk.add_(normals(seed, G_ID, m * j0, m * k, device).reshape(k, m), alpha=noise)
        At[j0 - lo:j1 - lo, :m] = blk
        b_part += blk.T @ x0[j0 - lo:j1 - lo]
        c[j0 - lo:j1 - lo] = blk @ y0 + z0[j0 - lo:j1 - lo] - q[j0 - lo:j1 - lo] * x0[j0 - lo:j1 - lo]
        del Ht, blk
    return Shard(m, n, lo, hi, lda, At, b_part, q, c, x0, y0, z0)


def shard_bounds(n: int, rank: int, world: int):
    """Contiguous column partition of [0, n) (rank r gets [n r / W, n (r+1) / W))."""
    return (n * rank) // world, (n * (rank + 1)) // world
