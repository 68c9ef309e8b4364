"""Seeded synthetic MNIST-shaped inputs, shared by the oracle tests, the GPU
parity tests and bench.py.

This module holds NO arithmetic of the method (no forward pass, no gradient,
no update, no averaging): it only draws inputs.  Both sides of every parity
test read the bytes it produces.

Stand-in for MNIST (§5.1: 28x28 grey images, 10 classes,
60,000 train / 10,000 test), which is not available in this container.
The recipe (BASELINE.json configs):

* class prototypes P_c, c = 0..9: a polyline of 3-5 control points drawn
  uniformly in the central box [4, 23]^2, with 12 Gaussian blobs
  (sigma = 1.5 px) placed evenly (by arc length) along it; P_c = min(1, sum of blobs);
* image i: y_i ~ Uniform{0..9};  x_i = clip(P_{y_i} + 0.1 * N(0, 1), 0, 1)   (fp32);
* rows are generated in chunks of CHUNK rows, chunk c of split s from its own
  PCG64 stream seeded by SeedSequence([seed, s, c]), so any row range can be
  regenerated without producing the rows before it (used by the full-size
  sampled parity tests).
"""
from .mnist_like import CHUNK, N_CLASSES, N_PIXELS, SIDE, prototypes, make_split, make_rows

__all__ = ["CHUNK", "N_CLASSES", "N_PIXELS", "SIDE", "prototypes", "make_split", "make_rows"]
