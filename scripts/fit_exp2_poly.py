"""Derivation of the frozen exp2_R coefficients (reading R3).

Lawson-reweighted least squares for a degree-5 relative-error minimax fit of 2^f on
[-1/2, 1/2], rounded to fp32.  The printed hex values are restated by hand in
oracle/bs_oracle.c and in the CUDA sources; this script is documentation of where they
came from, imported by neither side.
"""
import numpy as np

x = np.cos(np.linspace(0, np.pi, 4001)) * 0.5
f = np.exp2(x)
A = np.vander(x, 6, increasing=True) / f[:, None]
w = np.ones_like(x)
for _ in range(300):
    W = np.sqrt(w)
    c, *_ = np.linalg.lstsq(A * W[:, None], np.ones_like(x) * W, rcond=None)
    err = A @ c - 1
    w = w * np.abs(err)
    w /= w.sum()
print("max rel err (f64 coefficients):", np.abs(err).max())
for i, v in enumerate(c.astype(np.float32)):
    print(f"C{i} = {float(v).hex()}")
