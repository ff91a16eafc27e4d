"""Bank-conflict simulation of the bank-balanced CBSR entry order ("bank-balanced order").

The forward's NC = 16 layout puts copy q of column c at word 16 c + q, so its bank is q + 16 (c & 1); lane (s, p)
of an SW-lane sub-warp uses copy s*CPS + p % CPS, so lanes p and p + SW/2 of one edge share a copy and conflict
iff their two columns have the same parity.  In CBSR column order that happens for ~every instruction (2
wavefronts).  The banked order stores each row's even columns from the front and its odd columns from the back of
the priority list Q (first-half positions by group 0..3, then second-half positions by group 3..0), so a pair
differs in parity unless the row's even/odd split is unbalanced, and the unbalanced pairs land in group 3 first.

Prints the mean wavefronts per 32-lane RMW instruction (LDS or STS) for both orders, for the NC = 16 and the
NC = EPI (word EPI c + s) layouts, on N(0,1) rows (top-k column sets of H = 256)."""
import numpy as np

rng = np.random.default_rng(0)
H = 256


def rows(n, k):
    x = rng.standard_normal((n, H))
    return np.sort(np.argpartition(-x, k - 1, axis=1)[:, :k], axis=1)


def q_of(r, k):  # priority rank -> position (the forward's lane mapping: lane p, component e at 4 p + e)
    L = k // 8
    if r < k // 2:
        return 4 * (r % L) + r // L
    r2 = r - k // 2
    return 4 * (L + r2 % L) + 3 - r2 // L


def banked(idx):
    n, k = idx.shape
    out = np.empty_like(idx)
    for i in range(n):
        ev = idx[i][idx[i] % 2 == 0]
        od = idx[i][idx[i] % 2 == 1]
        for r, c in enumerate(ev):
            out[i, q_of(r, k)] = c
        for r, c in enumerate(od):
            out[i, q_of(k - 1 - r, k)] = c
    return out


def wavefronts(words):  # (m, 32) word addresses -> mean max distinct words per bank
    w = 0.0
    for a in words:
        d = {}
        for x in a:
            d.setdefault(x % 32, set()).add(x)
        w += max(len(s) for s in d.values())
    return w / len(words)


def sim(k, order, nc, n=3000):
    SW = k // 4 if k <= 128 else 32
    EPI = 32 // SW
    idx = rows(n * EPI, k)
    if order == "banked":
        idx = banked(idx)
    idx = idx.reshape(n, EPI, k)
    res = []
    for e in range(4):
        ent = np.array([4 * p + e for p in range(SW)])
        cols = idx[:, :, ent]  # n, EPI, SW
        s = np.arange(EPI)[None, :, None]
        p = np.arange(SW)[None, None, :]
        if nc == 16:
            cps = 16 // EPI
            words = 16 * cols + s * cps + p % cps
        else:  # NC = EPI
            words = EPI * cols + s
        res.append(wavefronts(words.reshape(n, 32)))
    return np.mean(res), res


if __name__ == "__main__":
    for k in (32, 64, 128):
        for nc in (16, "EPI"):
            a, _ = sim(k, "column", nc)
            b, per = sim(k, "banked", nc)
            print(f"k={k:3d} NC={nc!s:3}: column order {a:.2f}  banked {b:.2f}  (per group {' '.join('%.2f' % x for x in per)})")


def banked4(idx):
    """NC = 8 candidate (word 8 c + q, bank q + 8 (c mod 4)): lanes p = 2 m + pi of group e share copy pi with
    the other three lanes of the same pi; class m = c mod 4 takes slot m of the quads (e, pi) in priority order,
    the surplus fills the empty slots from the worst quad (group 3) back."""
    n, k = idx.shape
    quads = [(e, pi) for e in range(4) for pi in range(2)]
    out = np.empty_like(idx)
    for i in range(n):
        free = []
        surplus = []
        for m in range(4):
            cls = idx[i][idx[i] % 4 == m]
            for j, c in enumerate(cls):
                if j < 8:
                    e, pi = quads[j]
                    out[i, 4 * (2 * m + pi) + e] = c
                else:
                    surplus.append(c)
            for j in range(len(cls), 8):
                free.append((j, m))
        free.sort(key=lambda t: -t[0])  # worst quads first
        for c, (j, m) in zip(surplus, free):
            e, pi = quads[j]
            out[i, 4 * (2 * m + pi) + e] = c
    return out


def sim8(n=3000, k=32):
    EPI = 4
    idx = banked4(rows(n * EPI, k)).reshape(n, EPI, k)
    res = []
    for e in range(4):
        ent = np.array([4 * p + e for p in range(8)])
        cols = idx[:, :, ent]
        s = np.arange(EPI)[None, :, None]
        p = np.arange(8)[None, None, :]
        words = 8 * cols + s * 2 + p % 2
        res.append(wavefronts(words.reshape(n, 32)))
    return np.mean(res), res
