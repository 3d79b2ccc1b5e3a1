"""Shared helpers of the GPU parity tests (no method arithmetic: marshalling + comparisons)."""
import numpy as np


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def to_host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def assert_close(got, ref, tol, what=""):
    """Element-by-element |got - ref| <= tol * max|ref| (normwise-scaled elementwise test,
    DESIGN.md "Parity tolerances")."""
    scale = max(np.max(np.abs(ref)), 1e-300)
    err = np.max(np.abs(got - ref)) / scale if got.size else 0.0
    assert err <= tol, "%s: max|diff|/max|ref| = %.3e > %.1e" % (what, err, tol)
    return err


def sample_dofs(d, m, count, seed=0):
    """Structured + random samples: corners, boundary zones, tile edges, ragged tails."""
    rng = np.random.default_rng(seed)
    ns = m ** d
    idx = set()
    special = sorted(set([0, 1, 2, m // 2, m - 3, m - 2, m - 1, 31 % m, 32 % m, 127 % m, 128 % m]))
    special = [s for s in special if 0 <= s < m]
    for j in range(d):
        for _ in range(count // (2 * d) + 1):
            ks = [int(rng.choice(special)) for _ in range(d)]
            f = 0
            for k in ks:
                f = f * m + k
            idx.add(j * ns + f)
    while len(idx) < count:
        idx.add(int(rng.integers(0, d * ns)))
    return np.array(sorted(idx))
