"""Cases of the stage-level goldens (make_stage_golden.py) and of tests/test_gpu_stages.py.

A case is (kind, n, seed, BuildConfig kwargs): `kind` is a reference generator preset
(ingest.py:229-271) or one of the clouds below, built from numpy alone so the GPU box can
rebuild them without the reference."""
import numpy as np

STAGE_CASES = [
    ("uniform-cube", 20_000, 1, dict(T=1000)),
    ("stadium", 30_000, 3, dict(T=1500)),
    ("stadium", 200_000, 9, dict(T=300)),
    ("two-scans", 20_000, 4, dict(T=2000)),
    ("checker-plane", 10_000, 5, dict(T=800)),
    ("stadium", 100_000, 2, dict(T=400, initial_depth=6, extension_depth=3, max_depth=12)),
    ("stadium", 200_000, 9, dict(T=60)),
    ("identical", 2000, 0, dict(T=500)),
    ("blobs", 150_000, 11, dict(T=500)),
    ("blobs", 150_000, 12, dict(T=200, max_depth=14)),
]


def case_name(kind, n, seed, cfg):
    return f"{kind}_{n}_{seed}_" + "_".join(f"{k}{v}" for k, v in sorted(cfg.items()))


def custom_cloud(kind, n, seed):
    """(positions float64, colors uint8) of the non-preset kinds, else None.

    identical: n copies of one point (one extension chain down to max_depth);
    blobs: 7 tight gaussian clusters + a uniform background -- many overfull main cells with
    sibling and nested extension grids."""
    if kind == "identical":
        return np.tile(np.array([[0.25, 0.5, 0.75]]), (n, 1)), np.zeros((n, 3), np.uint8)
    if kind == "blobs":
        rng = np.random.default_rng(seed)
        k = 7
        centers = rng.random((k, 3)) * 0.8 + 0.1
        per = n // (k + 1)
        parts = [c + rng.normal(0.0, 4e-4 * (1 + j), (per, 3)) for j, c in enumerate(centers)]
        parts.append(rng.random((n - k * per, 3)))
        pos = np.concatenate(parts)[rng.permutation(n)]
        return pos, rng.integers(0, 256, (n, 3)).astype(np.uint8)
    return None
