"""Per-level cost of the cluster sweep on a synthetic level chain (run through the library's
ILU(0) apply on a lower-triangular matrix: L = its strict part, U = its diagonal).

Rows are level-major, R rows per level; row (l, i) reads E early sources (levels l-3..l-5),
M mid sources (level l-2) and T late sources (level l-1).  Per-level cost =
(t(L2) - t(L1)) / (L2 - L1) from the minimum of repeated applies."""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1808_08328_b200 import linalg  # noqa: E402

R = int(os.environ.get("SYN_R", 22))
E, M, T = (int(v) for v in os.environ.get("SYN_EMT", "21,3,3").split(","))


def matrix(L, seed=0):
    rng = np.random.default_rng(seed)
    n = L * R
    rows, cols = [], []
    for l in range(L):
        for i in range(R):
            r = l * R + i
            srcs = set()
            for d, k in ((1, T), (2, M)):
                if l - d >= 0:
                    srcs.update((l - d) * R + rng.choice(R, k, replace=False))
            if l - 3 >= 0:
                lo = max(0, l - 5) * R
                srcs.update(rng.choice(np.arange(lo, (l - 2) * R), min(E, (l - 2) * R - lo), replace=False))
            for c in sorted(srcs):
                rows.append(r); cols.append(c)
            rows.append(r); cols.append(r)
    vals = np.where(np.array(rows) == np.array(cols), 4.0, -1.0 / (E + M + T))
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def apply_time(L, reps=30):
    A = matrix(L)
    f = linalg.ilu0(A)
    b = np.ones(A.shape[0])
    z = linalg.apply_ilu0(f, b)
    ref = sp.linalg.spsolve_triangular(A, b, lower=True)
    err = np.abs(z - ref).max() / np.abs(ref).max()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        linalg.apply_ilu0(f, b)
        best = min(best, time.perf_counter() - t0)
    return best, err


L1, L2 = 500, 1500
t1, e1 = apply_time(L1)
t2, e2 = apply_time(L2)
print(f"R={R} E,M,T={E},{M},{T}: apply {t1 * 1e6:.0f} / {t2 * 1e6:.0f} us -> {(t2 - t1) / (L2 - L1) * 1e9:.0f} ns per level "
      f"({(t2 - t1) / (L2 - L1) * 1.965e9:.0f} cycles @1965 MHz); max rel err {max(e1, e2):.1e}")
