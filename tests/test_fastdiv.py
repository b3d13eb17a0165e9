"""The K1 key fast path (floor_div_pinned in k_frame.cu) must give floor(fl(x / r)) exactly (R5).
Re-derived here in IEEE float32 with numpy over adversarial and random values: whenever the fast
path answers, it equals floor of the correctly rounded quotient."""
import numpy as np


def fast_floor(x, r):
    x = np.asarray(x, np.float32)
    r = np.float32(r)
    rinv = np.float32(np.float32(1.0) / r)
    q = (x * rinv).astype(np.float32)
    fq = np.floor(q).astype(np.float32)
    d = (q - fq).astype(np.float32)
    tol = (np.abs(q) * np.float32(1e-6) + np.float32(1e-30)).astype(np.float32)
    fast = (d > tol) & (d < np.float32(1.0) - tol)
    exact = np.floor((x / r).astype(np.float32)).astype(np.float32)
    return fast, fq, exact


def test_fast_path_equals_pinned_floor():
    rng = np.random.default_rng(0)
    for r in [0.01, 0.02, 0.05, 0.1, 0.0123, 1.0, 3.7]:
        x = rng.uniform(-300, 300, 2_000_000).astype(np.float32)
        # adversarial: values within a few ulp of multiples of r
        k = rng.integers(-20000, 20000, 200_000).astype(np.float32)
        near = (k * np.float32(r)).astype(np.float32)
        jit = rng.integers(-8, 9, near.shape).astype(np.float32)
        near = np.nextafter(near, near + jit)  # a few ulp either side
        for xs in [x, near]:
            fast, fq, exact = fast_floor(xs, r)
            assert np.array_equal(fq[fast], exact[fast]), r
            assert fast.mean() > 0.5 or xs is near
