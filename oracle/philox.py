"""Philox4x32-10 counter-based RNG (Salmon et al., SC'11, "Parallel random
numbers: as easy as 1, 2, 3"), written out from the algorithm.

The paper fixes no RNG ("sampling input coordinates uniformly"); the
reading R8 in DESIGN.md picks Philox4x32-10 so that the GPU and this oracle
draw identical samples from independent implementations.

Pinned by tests/test_oracle_philox.py against the published Random123
known-answer vectors (tests/golden/philox_kat.txt).
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint64(0x9E3779B9)
W1 = np.uint64(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: (4, n) uint32-valued array-like, key: (2, n) or (2,) -> (4, n) uint32.

    One round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2;
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bump k += (W0, W1)
    between rounds; 10 rounds.
    """
    c = [np.asarray(x, dtype=np.uint64) & MASK32 for x in ctr]
    k0 = np.asarray(key[0], dtype=np.uint64) & MASK32
    k1 = np.asarray(key[1], dtype=np.uint64) & MASK32
    for r in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        if r < 9:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
    return np.stack([np.broadcast_to(x, np.broadcast(*c).shape) for x in c]).astype(np.uint32)


def stream_key(seed, stream):
    """Key for stream k: (seed_lo, seed_hi ^ k)  (R8: 0 init, 1 uniform,
    2 boundary, 4 decode queries)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return (seed & 0xFFFFFFFF, ((seed >> 32) ^ int(stream)) & 0xFFFFFFFF)


def u01(u):
    """uint32 -> float in [0, 1 - 2^-24]:  (u >> 8) * 2^-24, exact in float32."""
    return (np.asarray(u, dtype=np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
