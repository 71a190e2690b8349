"""ORACLE (test infrastructure only): shot sampling from a state vector.

SPEC `sample` (Fig. 3 caption, "10,000 measurements of the Bell state"):
i.i.d. draws of the basis index from |a_i|^2, deterministic given a seed. The plain definition is
inverse-CDF sampling: draw u ~ U[0,1), return the first index whose cumulative probability exceeds
u * total. Because floating point decides an integer here, this oracle fixes the uniform generator
and the summation order so that the library takes the same decisions:

  p_i   = re*re + im*im                        (numpy: two products, one sum; no FMA)
  S_b   = block sum over 2^lb1 logical indices: 32 lane sums (element 32k+l added sequentially in k),
          then halving (a[j] += a[j+h], h = 16, ..., 1)
  T_c   = sequential sum of the 2^lb2 block sums of superblock c; cum = sequential prefix of T
  u_s   = (splitmix64(seed + (s+1) * 0x9E3779B97F4A7C15) >> 11) * 2^-53,  t = u_s * cum[-1]
  search: first superblock with cum > t; running sum from cum[c-1] over its blocks -> first block
          with running > t; running sum from the value before that block over its p_i -> first
          index with running > t (ties to rounding: the last block / element with a nonzero sum).

Shares no code with the CUDA path. numpy's cumsum is a sequential running sum (no pairwise
reassociation), which is what makes the orders identical.
"""
from __future__ import annotations

import numpy as np

LB1 = 10
LB2 = 10
_M64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniforms(seed: int, shots: int) -> np.ndarray:
    return np.array([(splitmix64(seed + (s + 1) * 0x9E3779B97F4A7C15) >> 11) * 2.0 ** -53 for s in range(shots)])


def _lane_tree(x: np.ndarray) -> np.ndarray:
    """Halving reduction over the last axis of length 32: a[j] += a[j+h], h = 16..1."""
    a = x.copy()
    h = 16
    while h >= 1:
        a = a[..., :h] + a[..., h:2 * h]
        h //= 2
    return a[..., 0]


def block_sums(p: np.ndarray, n: int):
    lb1 = min(n, LB1)
    per = 1 << lb1
    nblk = 1 << (n - lb1)
    pb = p.reshape(nblk, per)
    if per >= 32:
        lanes = np.cumsum(pb.reshape(nblk, per // 32, 32), axis=1)[:, -1, :]    # sequential in k
    else:
        lanes = np.zeros((nblk, 32))
        lanes[:, :per] = pb
    return _lane_tree(lanes), lb1


def sample(psi: np.ndarray, shots: int, seed: int) -> np.ndarray:
    """psi in LOGICAL order (complex128, 2^n). Returns `shots` logical indices (uint64)."""
    n = int(psi.size).bit_length() - 1
    p = psi.real * psi.real + psi.imag * psi.imag
    S, lb1 = block_sums(p, n)
    nblk = S.size
    lb2 = min(n - lb1, LB2)
    nb = 1 << lb2
    nsup = nblk >> lb2
    T = np.cumsum(S.reshape(nsup, nb), axis=1)[:, -1]
    cum = np.cumsum(T)
    total = cum[-1]
    if not total > 0.0:
        raise ValueError("zero state")
    per = 1 << lb1
    out = np.empty(shots, dtype=np.uint64)
    for s, u in enumerate(uniforms(seed, shots)):
        t = u * total
        c = int(np.searchsorted(cum, t, side="right"))
        if c >= nsup:
            c = nsup - 1
            while c > 0 and cum[c] == cum[c - 1]:
                c -= 1
        start = cum[c - 1] if c else 0.0
        run = np.cumsum(np.concatenate([[start], S[c * nb:(c + 1) * nb]]))   # run[j+1] = after block j
        j = int(np.searchsorted(run[1:], t, side="right"))
        if j >= nb:                                    # rounding: last block with a nonzero sum
            nz = np.nonzero(S[c * nb:(c + 1) * nb] > 0.0)[0]
            j = int(nz[-1]) if nz.size else 0
        blk = c * nb + j
        pe = p[blk * per:(blk + 1) * per]
        run2 = np.cumsum(np.concatenate([[run[j]], pe]))
        i = int(np.searchsorted(run2[1:], t, side="right"))
        if i >= per:
            nz = np.nonzero(pe > 0.0)[0]
            i = int(nz[-1]) if nz.size else 0
        out[s] = (blk << lb1) | i
    return out
