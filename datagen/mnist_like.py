"""Synthetic MNIST-shaped data (see package docstring for the recipe).

No method arithmetic lives here; only seeded draws.
"""
from __future__ import annotations

import functools
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SIDE = 28
N_PIXELS = SIDE * SIDE          # 784 inputs
N_CLASSES = 10                  # 10 output neurons
CHUNK = 4096                    # rows per independently seeded chunk
NOISE_SIGMA = 0.1               # "N(0,0.1)" read as sigma = 0.1
BLOB_SIGMA = 1.5
N_BLOBS = 12
_SPLIT_ID = {"train": 0, "test": 1}
# "hard" variant for the §8(f) accuracy experiments only (the parity tests and benches use the
# default recipe): each image blends its prototype with another class's, x = (1-a)·P_y + a·P_y2
# + 0.35·N(0,1), a ~ U(0, 0.5), drawn from a separate stream so the default bytes are unchanged
HARD_SIGMA = 0.35
HARD_BLEND = 0.5


@functools.lru_cache(maxsize=8)
def prototypes(seed: int = 0) -> np.ndarray:
    """[10, 784] float32 class prototypes in [0, 1]."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 7777])))
    rr, cc = np.meshgrid(np.arange(SIDE, dtype=np.float64), np.arange(SIDE, dtype=np.float64),
                         indexing="ij")
    protos = np.zeros((N_CLASSES, N_PIXELS), dtype=np.float32)
    for c in range(N_CLASSES):
        n_ctrl = int(rng.integers(3, 6))
        ctrl = rng.uniform(4.0, 23.0, size=(n_ctrl, 2))
        seg = np.linalg.norm(np.diff(ctrl, axis=0), axis=1)
        cum = np.concatenate([[0.0], np.cumsum(seg)])
        total = cum[-1] if cum[-1] > 0 else 1.0
        img = np.zeros((SIDE, SIDE))
        for s in np.linspace(0.0, total, N_BLOBS):
            i = min(int(np.searchsorted(cum, s, side="right")) - 1, n_ctrl - 2)
            f = 0.0 if seg[i] == 0 else (s - cum[i]) / seg[i]
            p = ctrl[i] + f * (ctrl[i + 1] - ctrl[i])
            img += np.exp(-((rr - p[0]) ** 2 + (cc - p[1]) ** 2) / (2 * BLOB_SIGMA ** 2))
        protos[c] = np.minimum(1.0, img).astype(np.float32).reshape(-1)
    return protos


def _chunk(seed: int, split: int, c: int, protos: np.ndarray, hard: bool = False):
    if hard:
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, split, c, 1])))
        y = rng.integers(0, N_CLASSES, size=CHUNK, dtype=np.int32)
        y2 = (y + rng.integers(1, N_CLASSES, size=CHUNK, dtype=np.int32)) % N_CLASSES
        a = rng.uniform(0.0, HARD_BLEND, size=(CHUNK, 1)).astype(np.float32)
        x = rng.standard_normal((CHUNK, N_PIXELS), dtype=np.float32)
        x *= np.float32(HARD_SIGMA)
        x += (1.0 - a) * protos[y] + a * protos[y2]
        np.clip(x, 0.0, 1.0, out=x)
        return x, y
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, split, c])))
    y = rng.integers(0, N_CLASSES, size=CHUNK, dtype=np.int32)
    x = rng.standard_normal((CHUNK, N_PIXELS), dtype=np.float32)
    x *= np.float32(NOISE_SIGMA)
    x += protos[y]
    np.clip(x, 0.0, 1.0, out=x)
    return x, y


def make_rows(start: int, n: int, split: str = "train", seed: int = 0,
              out_x: np.ndarray | None = None, out_y: np.ndarray | None = None, hard: bool = False):
    """Rows [start, start+n) of a split: (X [n,784] float32, y [n] int32).

    Row r is always the same bytes regardless of which range asked for it.
    """
    sid = _SPLIT_ID[split]
    protos = prototypes(seed)
    x = out_x if out_x is not None else np.empty((n, N_PIXELS), dtype=np.float32)
    y = out_y if out_y is not None else np.empty((n,), dtype=np.int32)
    if n == 0:
        return x, y
    c0, c1 = start // CHUNK, (start + n - 1) // CHUNK

    def fill(c):
        cx, cy = _chunk(seed, sid, c, protos, hard)
        lo = max(start, c * CHUNK)
        hi = min(start + n, (c + 1) * CHUNK)
        x[lo - start:hi - start] = cx[lo - c * CHUNK:hi - c * CHUNK]
        y[lo - start:hi - start] = cy[lo - c * CHUNK:hi - c * CHUNK]

    chunks = range(c0, c1 + 1)
    if len(chunks) > 4:
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(fill, chunks))
    else:
        for c in chunks:
            fill(c)
    return x, y


def make_split(n: int, split: str = "train", seed: int = 0, hard: bool = False):
    """The first n rows of a split."""
    return make_rows(0, n, split, seed, hard=hard)
