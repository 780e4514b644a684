#!/usr/bin/env python
"""DRAM-traffic floors of the C2 step's 12 GEMM launches, against ncu.

For each launch (step order, as in profiles/r01_gemm_pair_ncu.md):
  * algorithmic  = (M K + K N + M N) * 2 B: every operand read once, C written once;
  * wave floor   = what the persistent kernel must read if the L2 keeps nothing
    across waves: the tile order of the scheduler (bands of GROUP_M 512-row
    tiles, M fastest; 74 CTA pairs -> 74 tiles in flight per wave), each wave
    streaming the K panels of its distinct A row-blocks and B column-blocks once,
    plus C.  When A + B fit in the L2 (<= 100 MB usable of 126 MB) the operands
    are read once instead.
  * measured     = dram__bytes_read.sum + dram__bytes_write.sum (ncu --set full,
    cold-cache replays), parsed from the summary table.

    python tools/traffic_model.py profiles/r01_gemm_pair_ncu.md
"""
import re
import sys

H, M_TOK = 4096, 16384
BM, BN, PAIRS, GROUP_M, L2_USABLE = 512, 256, 74, 8, 100e6


def c2_launches():
    h, m = H, M_TOK
    fwd = [("qkv fwd NN", m, 3 * h, h), ("proj fwd NN", m, h, h), ("fc1 fwd NN", m, 4 * h, h),
           ("fc2 fwd NN", m, h, 4 * h)]
    bwd = []
    for name, k, n in (("fc2", 4 * h, h), ("fc1", h, 4 * h), ("proj", h, h), ("qkv", h, 3 * h)):
        bwd.append((f"{name} dW TN", k, n, m))   # Gx = 1: dW first (axonn.cpp), then dI
        bwd.append((f"{name} dI NT", m, k, n))
    return fwd + bwd


def tile_coord(t, tiles_m, tiles_n, group_m):
    per = group_m * tiles_n
    g, r = divmod(t, per)
    first = g * group_m
    gm = min(tiles_m - first, group_m)
    return first + r % gm, r // gm


def wave_floor(M, N, K):
    tm, tn = -(-M // BM), -(-N // BN)
    a_bytes, b_bytes, c_bytes = 2 * M * K, 2 * K * N, 2 * M * N
    if a_bytes + b_bytes <= L2_USABLE:
        return a_bytes + b_bytes + c_bytes
    total = 0
    T = tm * tn
    for w0 in range(0, T, PAIRS):
        ms, ns = set(), set()
        for t in range(w0, min(T, w0 + PAIRS)):
            mi, ni = tile_coord(t, tm, tn, GROUP_M)
            ms.add(mi)
            ns.add(ni)
        rows = sum(min(BM, M - mi * BM) for mi in ms)
        cols = sum(min(BN, N - ni * BN) for ni in ns)
        total += 2 * K * (rows + cols)
    return total + c_bytes


def measured(md):
    out = []
    for line in open(md):
        f = [x.strip() for x in line.split("|")]
        if len(f) > 7 and re.fullmatch(r"\d+", f[1] or ""):
            out.append((float(f[5]) + float(f[6])) * 1e9)
    return out


def main(md):
    meas = measured(md)
    print("| launch | M×N×K | algorithmic GB | wave floor GB | measured GB | measured / floor |")
    print("|---|---|---|---|---|---|")
    ta = tf = tmz = 0.0
    for (name, M, N, K), mz in zip(c2_launches(), meas):
        alg = 2 * (M * K + K * N + M * N)
        fl = wave_floor(M, N, K)
        ta, tf, tmz = ta + alg, tf + fl, tmz + mz
        print(f"| {name} | {M}×{N}×{K} | {alg / 1e9:.3f} | {fl / 1e9:.3f} | {mz / 1e9:.3f} | {mz / fl:.2f} |")
    n = len(meas)
    print(f"| **per launch (mean of {n})** | | {ta / n / 1e9:.3f} | {tf / n / 1e9:.3f} | "
          f"{tmz / n / 1e9:.3f} | {tmz / tf:.2f} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_gemm_pair_ncu.md")
