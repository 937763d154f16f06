"""Canonical seeded generators for BASELINE.json configs; synthetic stand-ins
with the configs' shapes, sizes and value distributions (no public dataset is used)."""
import numpy as np


def make_config(name: str, n_override=None):
    if name == "cfg1":
        rng = np.random.default_rng(0)
        n = n_override or 10000
        X = rng.standard_normal((n, 32), dtype=np.float32)
        A = rng.integers(1, 5, (n, 1), dtype=np.int32)
        QX = rng.standard_normal((200, 32), dtype=np.float32)
        QA = rng.integers(1, 5, (200, 1), dtype=np.int32)
        return X, A, QX, QA, (4,)
    if name == "cfg2":
        # N=1M, d=128, integers 0..255 as fp32: 1000 Gaussian centres U[0,255]^128 (literal
        # reading), sigma=20, rounded + clipped; 3 attributes (3/5/10) uniform; 10k queries
        # drawn the same way with a full 3-attribute constraint.
        rng = np.random.default_rng(0)
        n = n_override or 1_000_000
        q = 10_000
        centres = rng.uniform(0, 255, (1000, 128))
        def draw(cnt):
            lab = rng.integers(0, 1000, cnt)
            out = np.empty((cnt, 128), np.float32)
            for b in range(0, cnt, 65536):
                e = min(cnt, b + 65536)
                x = centres[lab[b:e]] + 20.0 * rng.standard_normal((e - b, 128))
                out[b:e] = np.clip(np.rint(x), 0, 255)
            return out
        X = draw(n)
        A = np.stack([rng.integers(1, c + 1, n) for c in (3, 5, 10)], 1).astype(np.int32)
        QX = draw(q)
        QA = np.stack([rng.integers(1, c + 1, q) for c in (3, 5, 10)], 1).astype(np.int32)
        return X, A, QX, QA, (3, 5, 10)
    raise ValueError(name)
