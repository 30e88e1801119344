"""CPU simulation of K2c/K2d's query-block pairing on one head's real plan
(oracle routing of the generator's data, Wan2.1-14B shape): union tiles per
k of consecutive pairs, of the shipped window (+-48 blocks, 16 candidates,
overlap desc / index asc) and of variants -- wider windows, more candidates,
a full O(N^2) candidate search, nearest-first tie-breaking.

    python tools/sim_pairing.py [sparsity]       (~10 s per data kind)

Results: profiles/r02n_pairing_sim.log."""
import sys
import time

import numpy as np

sys.path.insert(0, '/root/repo')
import oracle as O
L, d, r = 75600, 128, float(sys.argv[1]) if len(sys.argv) > 1 else 0.875
res = {}
for kind in ("gaussian", "clustered"):
    t=time.time()
    q, k, v = O.gen(kind, 0, 1, L, d)
    kbar = O.block_stats(k[0], v[0])[0]
    qb = O.query_means(q[0])
    N = qb.shape[0]; kk = O.sparsity_to_k(r, N)[0]
    sel = O.select_plain(qb, kbar, kk, d ** -0.5)
    M = np.zeros((N, N), np.int32); M[np.arange(N)[:, None], sel] = 1
    ov = M @ M.T
    np.fill_diagonal(ov, -1)
    def cands(win, kc=16, near=False):
        C = []
        for i in range(N):
            lo, hi = (max(0, i - win), min(N, i + win + 1)) if win else (0, N)
            js = [j for j in range(lo, hi) if j != i]
            js.sort(key=(lambda j: (-ov[i, j], abs(i - j), j)) if near else (lambda j: (-ov[i, j], j)))
            C.append(js[:kc])
        return C
    def match(C):
        partner = [-1] * N
        for rnd in range(64):
            prop = [-1] * N
            for i in range(N):
                if partner[i] < 0:
                    for j in C[i]:
                        if partner[j] < 0:
                            prop[i] = j; break
            prog = False
            for i in range(N):
                j = prop[i]
                if j >= 0 and prop[j] == i:
                    partner[i] = j; prog = True
            if not prog: break
        pairs, pend = [], -1
        for i in range(N):
            j = partner[i]
            if j > i: pairs.append((i, j))
            elif j < 0:
                if pend < 0: pend = i
                else: pairs.append((pend, i)); pend = -1
        if pend >= 0: pairs.append((pend, -1))
        return pairs
    def union(pairs):
        u = 0
        for a, b in pairs:
            u += kk if b < 0 else 2 * kk - (ov[a, b])
        return u / (len(pairs) * kk)
    cons = [(2 * t, 2 * t + 1 if 2 * t + 1 < N else -1) for t in range((N + 1) // 2)]
    print(kind, "N", N, "k", kk, "consecutive", round(union(cons), 4),
          "win48", round(union(match(cands(48))), 4), "win96", round(union(match(cands(96))), 4),
          "full16", round(union(match(cands(0))), 4), "full32", round(union(match(cands(0, 32))), 4), "full64", round(union(match(cands(0, 64))), 4), "win48c32", round(union(match(cands(48, 32))), 4), "full16near", round(union(match(cands(0, 16, True))), 4), "full32near", round(union(match(cands(0, 32, True))), 4), "win48near", round(union(match(cands(48, 16, True))), 4), round(time.time()-t,1), "s", flush=True)
