"""Shared-memory wavefronts of BS6's row-sum reads and value-tile stores for
candidate value-tile layouts (CPU model of scripts/expt + sb_gs_pipe.cu).

Model: a warp's 8-byte shared access costs max over the 16 bank pairs of the
number of distinct 8-byte words it touches there (>= 2 for 32 lanes).
Rows of a super-block are owned by thread t = row % 128 (warp = 32 rows);
iteration c of the row loop has every lane with c < len read entry start+c.
"""
import sys

import numpy as np


def row_lengths(K, p):
    g = K * p + 1
    a = np.arange(g)
    cnt = np.where((a % p == 0) & (a > 0) & (a < K * p), 2, 1)
    return (cnt[None, None, :] * cnt[None, :, None] * cnt[:, None, None]).reshape(-1)


def superblocks(rs, npb=512):
    ng = len(rs) - 1
    out, r = [], 0
    while r < ng:
        lim = rs[r] + npb
        j = np.searchsorted(rs, lim, side="right") - 1
        j = max(j, r + 1)
        out.append((r, j))
        r = j
    return out


LAYOUTS = {
    "csr": lambda k, j, P: k,
    "xor4": lambda k, j, P: k ^ ((k >> 4) & 15),
    "pad16": lambda k, j, P: k + (k >> 4),
    "xor3": lambda k, j, P: k ^ ((k >> 3) & 15),
    "rowshift": lambda k, j, P: k + j,
}


def wavefronts(addrs):
    if len(addrs) == 0:
        return 0
    words = np.unique(addrs)
    return max(2 if len(addrs) > 16 else 1, np.bincount(words % 16, minlength=16).max())


def sim(K, p, maxsb=4000):
    L = row_lengths(K, p)
    rs = np.concatenate([[0], np.cumsum(L)])
    sbs = superblocks(rs)[:maxsb]
    res = {name: [0, 0] for name in list(LAYOUTS) + ["transposed"]}
    for r0, r1 in sbs:
        e0 = rs[r0]
        starts = rs[r0:r1] - e0
        lens = L[r0:r1]
        nrows = r1 - r0
        ne = rs[r1] - e0
        rowid = np.repeat(np.arange(nrows), lens)
        kin = np.arange(ne) - starts[rowid]
        P = nrows | 1
        for name, f in LAYOUTS.items():
            slot = np.array([f(int(k), int(j), P) for k, j in zip(range(ne), rowid)])
            # stores: consecutive entries per warp instruction (lanes = entries)
            for w in range(0, ne, 32):
                res[name][1] += wavefronts(slot[w:w + 32])
            for w in range(0, nrows, 32):
                rows = np.arange(w, min(w + 32, nrows))
                for c in range(lens[rows].max()):
                    act = rows[lens[rows] > c]
                    res[name][0] += wavefronts(slot[starts[act] + c])
        # transposed: entry (j, k) at k * P + j
        tslot = kin * P + rowid
        for w in range(0, ne, 32):
            res["transposed"][1] += wavefronts(tslot[w:w + 32])
        for w in range(0, nrows, 32):
            rows = np.arange(w, min(w + 32, nrows))
            for c in range(lens[rows].max()):
                act = rows[lens[rows] > c]
                res["transposed"][0] += wavefronts(c * P + act)
    return len(sbs), res


for N in [int(v) for v in (sys.argv[1:] or ["1", "2", "3", "5", "7"])]:
    K = max(4, int(round((2e5 ** (1 / 3) - 1) / N)))
    nsb, res = sim(K, N, maxsb=600)
    base = sum(res["csr"])
    print(f"N={N} K={K} superblocks={nsb}: (row-sum reads, tile stores, total vs csr)")
    for name, (rd, stv) in res.items():
        print(f"   {name:10s} {rd:8d} {stv:8d}  {(rd + stv) / base:.2f}")
