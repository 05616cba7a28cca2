"""Pin the OpenBLAS summation order the degree decision depends on
(oracle/blasorder.c) to numpy itself, on the build host that recorded the
reference goldens (numpy 2.3.5, scipy-openblas 0.3.30, kernel SkylakeX, 8
threads).  Writes tests/golden/blas_order.npz: for seeded random vectors the
value of numpy's x.dot(y) (np.linalg.norm's sum, polyprec.py:46-51), and for
seeded tall matrices numpy's A.T @ A (the syrk of polyprec.py:118).  Inputs
are regenerated from the seeds (numpy PCG64 is stable), so the fixture is
small.

    python tests/golden/make_blas_golden.py
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

DOT_CASES = [(s, n) for s, n in enumerate(
    [1, 15, 16, 17, 31, 32, 33, 48, 100, 377, 1000, 1728, 4096, 5000, 9999, 10000, 10001,
     12345, 65536, 100003, 262147, 1000000])]
GRAM_CASES = [(100 + s, n, k) for s, (n, k) in enumerate(
    [(200, 5), (384, 7), (767, 9), (768, 11), (1151, 13), (4096, 17), (5000, 23), (12345, 27)])]


def dot_inputs(seed, n):
    g = np.random.default_rng(seed)
    x = g.uniform(-1, 1, n) * 10.0 ** g.uniform(-2, 2)
    y = x if seed % 3 == 0 else g.uniform(-1, 1, n)
    return x, y


def gram_input(seed, n, k):
    g = np.random.default_rng(seed)
    # columns of very different scales, like a power basis
    return g.uniform(-1, 1, (n, k)) * 10.0 ** g.uniform(-3, 3, k)


def main():
    from threadpoolctl import threadpool_info
    info = [i for i in threadpool_info() if i.get("internal_api") == "openblas"]
    out = {}
    out["dot_cases"] = np.array(DOT_CASES, dtype=np.int64)
    out["dot_values"] = np.array([np.dot(*dot_inputs(s, n)) for s, n in DOT_CASES])
    out["gram_cases"] = np.array(GRAM_CASES, dtype=np.int64)
    for s, n, k in GRAM_CASES:
        P = np.zeros((n, k + 2))
        P[:, 1:k + 1] = gram_input(s, n, k)
        AV = P[:, 1:k + 1]  # the same strided view numpy sees in polyprec.py:118
        out[f"gram_{s}"] = AV.T @ AV
    out["openblas"] = np.array(str(info))
    np.savez_compressed(os.path.join(HERE, "blas_order.npz"), **out)
    print("wrote", len(out), "arrays;", info)


if __name__ == "__main__":
    main()
