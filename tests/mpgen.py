"""Test-input construction helpers (vectorised numpy; exact by construction)."""
from __future__ import annotations

import numpy as np

EXP_ZERO = -(1 << 31)


def clear_below(limbs: np.ndarray, bits: int) -> np.ndarray:
    """Zero every bit below precision `bits` in left-aligned (L, N) limbs."""
    L = limbs.shape[0]
    sh = 32 * L - bits
    out = limbs.copy()
    for k in range(L):
        lo, hi = 32 * k, 32 * k + 32
        if hi <= sh:
            out[k] = 0
        elif lo < sh:
            out[k] &= np.uint32((0xFFFFFFFF << (sh - lo)) & 0xFFFFFFFF)
    return out


def random_mantissas(rng: np.random.Generator, L: int, n: int, bits: int) -> np.ndarray:
    m = rng.integers(0, 1 << 32, size=(L, n), dtype=np.uint64).astype(np.uint32)
    m[L - 1] |= np.uint32(0x80000000)
    return clear_below(m, bits)


def structured_pairs(rng: np.random.Generator, L: int, n: int, bits: int):
    """x, y operand arrays (limbs, exp, sign) stressing alignment / cancellation /
    ties / zeros for add, sub, mul and div."""
    xm = random_mantissas(rng, L, n, bits)
    ym = random_mantissas(rng, L, n, bits)
    xe = rng.integers(-40, 40, size=n).astype(np.int64)
    # exponent gaps around every boundary the add kernel has
    gaps = np.array([0, 1, 2, 3, 31, 32, 33, 63, 64, 65, bits - 2, bits - 1, bits, bits + 1, bits + 2,
                     32 * L - 1, 32 * L, 32 * L + 1, 32 * L + 31, 32 * L + 32, 32 * L + 33, 32 * L + 64,
                     32 * L + 100, 5000], dtype=np.int64)
    kind = rng.integers(0, 4, size=n)
    d = np.where(kind == 0, rng.integers(0, 8, size=n),
                 np.where(kind == 1, gaps[rng.integers(0, len(gaps), size=n)],
                          rng.integers(0, 32 * L + 70, size=n)))
    d = np.where(rng.random(n) < 0.5, d, -d)
    ye = xe - d
    xs = rng.integers(0, 2, size=n).astype(np.uint8)
    ys = rng.integers(0, 2, size=n).astype(np.uint8)
    # special mantissas
    sel = rng.random(n)
    same = sel < 0.08                      # y mantissa == x mantissa (exact cancellation / doubling)
    ym[:, same] = xm[:, same]
    ones = (sel >= 0.08) & (sel < 0.14)   # all ones at p bits (carry chains)
    ym[:, ones] = clear_below(np.full((L, int(ones.sum())), 0xFFFFFFFF, np.uint32), bits)
    pow2 = (sel >= 0.14) & (sel < 0.20)   # 1000..0 (power of two)
    ym[:, pow2] = 0
    ym[L - 1, pow2] = 0x80000000
    xpow2 = (sel >= 0.20) & (sel < 0.26)
    xm[:, xpow2] = 0
    xm[L - 1, xpow2] = 0x80000000
    # near-equal: y = x +- 1 ulp (massive cancellation)
    near = (sel >= 0.26) & (sel < 0.32)
    ym[:, near] = xm[:, near]
    ye[near] = xe[near]
    sh = 32 * L - bits
    lsb = np.uint64(1) << np.uint64(sh % 32)
    k0 = sh // 32
    ym[k0, near] = (ym[k0, near].astype(np.uint64) ^ lsb).astype(np.uint32)
    ym[L - 1, near] |= np.uint32(0x80000000)
    # sparse x (top bit + one more bit) times y with boundary-valued low limbs: puts
    # the product's guard limb on / next to the rounding boundaries, exercising the
    # short-product decision and its full-product fallback in mp_mul
    sparse = (sel >= 0.32) & (sel < 0.40)
    ns = int(sparse.sum())
    xm[:, sparse] = 0
    xm[L - 1, sparse] = 0x80000000
    pos = rng.integers(0, 32 * L - 1, size=ns)
    cols = np.nonzero(sparse)[0]
    for c, p_ in zip(cols, pos):
        if p_ >= 32 * L - bits:
            xm[p_ // 32, c] |= np.uint32(1 << (p_ % 32))
    bvals = np.array([0, 1, 2, 0x7FFFFFFF, 0x80000000, 0x80000001, 0xFFFFFFFE, 0xFFFFFFFF, 0x7FFFFFF0,
                      0x8000000F], np.uint64)
    for k in range(L):
        ym[k, sparse] = bvals[rng.integers(0, len(bvals), size=ns)].astype(np.uint32)
    ym[L - 1, sparse] |= np.uint32(0x80000000)
    ym[:, sparse] = clear_below(ym[:, sparse], bits)
    # zeros of both signs
    zx = rng.random(n) < 0.03
    zy = rng.random(n) < 0.03
    xm[:, zx] = 0
    ym[:, zy] = 0
    xe = np.where(zx, EXP_ZERO, xe).astype(np.int32)
    ye = np.where(zy, EXP_ZERO, ye).astype(np.int32)
    return (xm, xe, xs), (ym, ye, ys)


def tie_cases(L: int, bits: int):
    """x + y exactly halfway between two p-bit numbers (round-to-even checks)."""
    xs, ys = [], []
    for lsb_odd in (0, 1):
        for sgn in (0, 1):
            xm = np.zeros(L, np.uint32)
            xm[L - 1] = 0x80000000
            if lsb_odd:
                sh = 32 * L - bits
                xm[sh // 32] |= np.uint32(1 << (sh % 32))
            # x = 0.1xxx * 2^1 ; y = 2^(1 - bits - 1) = half an ulp of x
            xs.append((xm, 1, sgn))
            ym = np.zeros(L, np.uint32)
            ym[L - 1] = 0x80000000
            ys.append((ym, 1 - bits, sgn))
    def pack(items):
        m = np.stack([i[0] for i in items], axis=1)
        e = np.array([i[1] for i in items], np.int32)
        s = np.array([i[2] for i in items], np.uint8)
        return m, e, s
    return pack(xs), pack(ys)


def carry_patterns(L: int, bits: int) -> np.ndarray:
    """(L, P) mantissas that maximise / isolate the carries of the limb-product chains:
    all ones, a single saturated limb at every position, alternating saturated limbs, ..."""
    cols = []
    full = np.full(L, 0xFFFFFFFF, np.uint64)
    cols.append(full.copy())
    cols.append(np.full(L, 0xFFFFFFFE, np.uint64))
    top = np.zeros(L, np.uint64)
    top[L - 1] = 0x80000000
    cols.append(top.copy())
    t = full.copy()
    t[L - 1] = 0x80000000
    cols.append(t)
    t = np.zeros(L, np.uint64)
    t[L - 1] = 0xFFFFFFFF
    cols.append(t)
    for par in (0, 1):
        t = np.zeros(L, np.uint64)
        t[par::2] = 0xFFFFFFFF
        cols.append(t)
    for k in range(L):
        t = np.zeros(L, np.uint64)
        t[k] = 0xFFFFFFFF
        cols.append(t)
        t = full.copy()
        t[k] = 0
        cols.append(t)
    m = np.stack(cols, axis=1).astype(np.uint32)
    m[L - 1] |= np.uint32(0x80000000)
    return clear_below(m, bits)
