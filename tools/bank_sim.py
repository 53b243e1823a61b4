"""Shared-memory bank-conflict model of the Stockham exchange layouts (design aid, no GPU).

wavefronts(instr) = max over the 32 4-byte banks of the number of distinct 4-byte words a
warp touches in that bank (Volta+ model); ideal = warp bytes / 128.  Mirrors the index maps
in paper_2601_12209_b200/csrc/fft_kernels.cuh (sidx_contig / sidx_strided).
"""
import sys
from itertools import product


def schedule(n, dp):
    rads = []
    m = n
    for p in (7, 5, 3):
        while m % p == 0:
            rads.append(p); m //= p
    pw = []
    while m % 16 == 0:
        pw.append(16); m //= 16
    if m > 1:
        pw.append(m)
    return pw + rads  # radix-2^k passes first, odd radices last


def wavefronts(words_per_lane):
    """Accesses wider than 4 B are split into phases of 128 B worth of lanes (half-warps for
    8 B, quarter-warps for 16 B, as measured by ncu on B200); within a phase the wavefront count
    is the max number of distinct words on one bank."""
    per = len(words_per_lane[0]) if words_per_lane else 1
    lanes_per_phase = 32 // per
    tot = 0
    for p0 in range(0, len(words_per_lane), lanes_per_phase):
        banks = {}
        for ws in words_per_lane[p0:p0 + lanes_per_phase]:
            for w in ws:
                banks.setdefault(w % 32, set()).add(w)
        tot += max(len(s) for s in banks.values())
    return tot


def sim(n, dp, fam, W=None, padshift=None):
    es = 16 if dp else 8
    rads = schedule(n, dp)
    T = n // max(rads)
    tot = ideal = 0
    Ns = 1
    if fam == "contig":
        lpc = max(1, 256 // T)
        LS = n + (n >> padshift) + (2 if dp else 1) * 0
        def addr(line, t): return line * LS + t + (t >> padshift)
        nthreads = T * lpc
        def lane_info(tid): return tid // T, tid % T  # (line, j)
    else:
        nthreads = T * W
        R0 = rads[0]
        def addr(c, t): return t * W + c + (t // R0) * padshift
        def lane_info(tid): return tid % W, tid // W
    for p, R in enumerate(rads):
        nb = n // R
        for u in range((nb + T - 1) // T):
            for phase in ("read", "write"):
                if phase == "read" and p == 0: continue
                if phase == "write" and p == len(rads) - 1: continue
                for r in range(R):
                    for w0 in range(0, nthreads, 32):
                        lanes = []
                        for tid in range(w0, w0 + 32):
                            a, j = lane_info(tid)
                            b = j + T * u
                            if b >= nb: continue
                            if phase == "read": t = b + r * nb
                            else: t = (b // Ns) * Ns * R + b % Ns + r * Ns
                            e = addr(a, t)
                            lanes.append([e * es // 4 + q for q in range(es // 4)])
                        if not lanes: continue
                        tot += wavefronts(lanes)
                        ideal += max(1, (len(lanes) * es + 127) // 128)
        Ns *= R
    return tot / max(ideal, 1), rads, T


if __name__ == "__main__":
    for dp in (False, True):
        for n in [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 96, 192, 384, 768, 1536]:
            res = []
            for ps in (3, 4, 5):
                res.append(("c%d" % ps, round(sim(n, dp, "contig", padshift=ps)[0], 2)))
            for W in ((4, 8) if dp else (8, 16)):
                for pad in (0, W // 2, W, 2 * W):
                    res.append(("s%d/%d" % (W, pad), round(sim(n, dp, "strided", W=W, padshift=pad)[0], 2)))
            print("dp" if dp else "sp", n, schedule(n, dp), res)
