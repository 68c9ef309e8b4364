"""The seeded input generator (datagen/): row-range independence, the default recipe's
bytes pinned (every parity fixture and bench depends on them), and the §8(f) "hard"
variant drawn from a separate stream."""
import hashlib

import numpy as np

from datagen import CHUNK, make_rows, make_split


def _h(x, y):
    return hashlib.sha256(x.tobytes() + y.tobytes()).hexdigest()


def test_default_bytes_pinned():
    x, y = make_rows(CHUNK - 6, 20, "train", 0)      # straddles a chunk boundary
    assert _h(x, y) == "bab97d2cd91774921306aa5f2a43463dc64e6b99fa48658f707dd1282ce1d0b4"


def test_row_ranges_agree():
    X, y = make_split(CHUNK + 50, "train", 0)
    x2, y2 = make_rows(CHUNK - 10, 40, "train", 0)
    np.testing.assert_array_equal(X[CHUNK - 10:CHUNK + 30], x2)
    np.testing.assert_array_equal(y[CHUNK - 10:CHUNK + 30], y2)


def test_hard_variant_separate():
    x, y = make_split(200, "test", 0)
    xh, yh = make_split(200, "test", 0, hard=True)
    assert not np.array_equal(x, xh)
    assert xh.min() >= 0.0 and xh.max() <= 1.0 and set(np.unique(yh)) <= set(range(10))
    x2, y2 = make_split(200, "test", 0)
    np.testing.assert_array_equal(x, x2)              # the default is untouched by the variant
