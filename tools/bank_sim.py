"""Shared-memory bank-conflict model of K_A4's access patterns (tools only; used to pick the
padded row strides). Model: 32 banks x 4 B; a warp access of w bytes/thread is split into
phases of 128/w threads; a phase costs max over banks of the distinct 4-byte words it touches.
"""
import itertools
import sys


def wavefronts(addrs_bytes, width):
    """addrs_bytes: list of 32 byte addresses (None = inactive lane)."""
    per = 128 // width if width >= 4 else 32
    per = min(per, 32) if width <= 4 else per
    if width <= 4:
        per = 32
    tot = 0
    for p0 in range(0, 32, per):
        banks = {}
        for a in addrs_bytes[p0:p0 + per]:
            if a is None:
                continue
            for wd in range(max(width // 4, 1)):
                word = a // 4 + wd
                banks.setdefault(word % 32, set()).add(word)
        if banks:
            tot += max(len(v) for v in banks.values())
    return tot


def ideal(addrs_bytes, width):
    n = len({a for a in addrs_bytes if a is not None})
    return max(1, (n * width + 127) // 128) if n else 0


def pattern_cost(fn, nthreads, width):
    """fn(t) -> list of byte addresses accessed by thread t (one per 'instruction' index)."""
    per_t = [fn(t) for t in range(nthreads)]
    ninst = max(len(x) for x in per_t)
    w = i = 0
    for warp in range((nthreads + 31) // 32):
        for k in range(ninst):
            addrs = []
            for lane in range(32):
                t = warp * 32 + lane
                addrs.append(per_t[t][k] if t < nthreads and k < len(per_t[t]) else None)
            if any(a is not None for a in addrs):
                w += wavefronts(addrs, width)
                i += ideal(addrs, width)
    return w, i


def ka4(WP, WI, WK, WM, TO, QS, verbose=False):
    D = 8  # bytes per double
    res = {}

    def s1(t):  # 19 pairs x 13 strips x 3 rows: p rows (2 x ld2), I (ld2), stores
        if t >= 19 * 13:
            return []
        xp, y0 = 2 * (t % 19), 3 * (t // 19)
        out = []
        for i in range(3):
            y = y0 + i
            if y >= WI_ROWS:
                continue
            out += [((y + 2) * WP + xp) * D, ((y + 2) * WP + xp + 2) * D, (y * WI + xp) * D]
        return out
    WI_ROWS, WK_ROWS, WM_ROWS = 38, 36, 34
    res["S1 ld p/I"] = pattern_cost(s1, 256, 16)
    res["S1 st s"] = pattern_cost(lambda t: [((3 * (t // 19) + i) * WI + 2 * (t % 19)) * D for i in range(3)
                                              if t < 247 and 3 * (t // 19) + i < 38], 256, 16)

    def s2(t):
        if t >= 18 * 14:
            return []
        xp, y0 = 2 * (t % 18), 3 * (t // 18)
        out = []
        for i in range(3):
            y = y0 + i
            if y >= 36:
                continue
            out += [((y + 2) * WI + xp) * D, ((y + 2) * WI + xp + 2) * D, (y * WK + xp) * D]
        return out
    res["S2 ld s/mu"] = pattern_cost(s2, 256, 16)

    def s3(t):
        if t >= 17 * 15:
            return []
        xp, y0 = 2 * (t % 17), 3 * (t // 17)
        out = []
        for i in range(3):
            y = y0 + i
            if y >= 34:
                continue
            out += [((y + 2) * WK + xp) * D, ((y + 2) * WK + xp + 2) * D, ((y + 2) * WI + xp + 2) * D,
                    (y * WM + xp) * D]
        return out
    res["S3 ld a/s st M"] = pattern_cost(s3, 256, 16)

    def s5(t):
        xp, y0 = 2 * (t & 15), 2 * (t >> 4)
        out = []
        for i in range(2):
            y = y0 + i
            out += [((y + 2) * WM + xp) * D, ((y + 2) * WM + xp + 2) * D, (y * TO + xp) * D]
        return out
    res["S5 ld M/O"] = pattern_cost(s5, 256, 16)

    def pown(t):
        return [((2 * (t >> 4) + i + 4) * WP + 2 * (t & 15) + 4) * D for i in range(2)]
    res["pown"] = pattern_cost(pown, 256, 16)

    def s4q(t):  # data term q loads (CF = 4, DM = 5)
        Jc, rest = t % 8, t // 8
        Ic0 = (rest % 2) * 4
        return [((Ic0 + m) * QS + Jc + b) * D for m in range(8) for b in range(5)]
    res["S4 q"] = pattern_cost(s4q, 256, 8)

    def s4o(t):
        Jc, rest = t % 8, t // 8
        Ic0, ph = (rest % 2) * 4, rest // 2
        pr, pc = ph // 4, ph % 4
        return [(((Ic0 + k) * 4 + pr) * TO + Jc * 4 + pc) * D for k in range(4)]
    res["S4 st O"] = pattern_cost(s4o, 256, 8)
    tw = sum(v[0] for v in res.values())
    ti = sum(v[1] for v in res.values())
    if verbose:
        for k, v in res.items():
            print(f"  {k:16s} {v[0]:6d} / ideal {v[1]:6d}")
    return tw, ti


if __name__ == "__main__":
    base = dict(WP=40, WI=38, WK=36, WM=34, TO=32, QS=24)
    print("current", ka4(**base, verbose=True))
    best = None
    for WP, WI, WK, WM, TO in itertools.product(range(40, 50, 2), range(38, 48, 2), range(36, 46, 2),
                                                range(34, 44, 2), range(32, 42, 2)):
        c = ka4(WP, WI, WK, WM, TO, 24)[0]
        if best is None or c < best[0]:
            best = (c, WP, WI, WK, WM, TO)
    print("best strides", best)
    for QS in range(14, 34):
        print("QS", QS, ka4(*best[1:], QS)[0])


def coord_search(start, lo=32, hi=60):
    cur = dict(start)
    best = ka4(**cur)[0]
    improved = True
    while improved:
        improved = False
        for k in ("WP", "WI", "WK", "WM", "TO"):
            floor = {"WP": 40, "WI": 38, "WK": 36, "WM": 34, "TO": 32}[k]
            for v in range(floor, hi + 1, 2):
                trial = dict(cur, **{k: v})
                c = ka4(**trial)[0]
                if c < best or (c == best and v < cur[k]):
                    if c < best:
                        improved = True
                    best, cur = c, trial
    return best, cur
