"""State digests for parity fixtures at config size (test infrastructure).

A full 2^20..2^24-amplitude state is too large to commit, so the fixtures made by
`make_config_goldens.py` from the REAL reference store a digest that the GPU tests
recompute from the device state and compare at the north_star tolerance:

* `amps`   -- the amplitudes at 512 fixed indices (seeded choice over [0, 2^n));
* `p1`     -- per-qubit marginals P(q = 1) = sum |psi_i|^2 over i with bit q set;
* `proj`   -- <r_k|psi> for 4 fixed unit vectors with components ±2^{-n/2} (signs from a
              seeded generator), i.e. every amplitude enters every projection;
* `norm2`  -- sum |psi_i|^2.

All inputs are numpy arrays; the sign vectors and indices are regenerated from fixed
seeds with numpy's PCG64 (identical on every host), so nothing but the digest travels.
"""

from __future__ import annotations

import numpy as np

N_IDX = 512
N_PROJ = 4


def indices(n: int) -> np.ndarray:
    size = 1 << n
    k = min(N_IDX, size)
    return np.sort(np.random.default_rng(777 + n).choice(size, k, replace=False))


def sign_vector(n: int, k: int) -> np.ndarray:
    bits = np.random.default_rng(1000 + 31 * n + k).integers(0, 4, 1 << n, dtype=np.int8)
    re = np.where(bits & 1, -1.0, 1.0)
    im = np.where(bits & 2, -1.0, 1.0)
    return (re + 1j * im) * (0.5 ** ((n + 1) / 2))


def digest(amps: np.ndarray, n: int) -> dict:
    psi = np.asarray(amps, dtype=np.complex128)
    assert psi.shape == (1 << n,)
    prob = psi.real * psi.real + psi.imag * psi.imag
    idx = indices(n)
    p1 = []
    view = prob.reshape((2,) * n)  # axis a <-> qubit n-1-a (little-endian index)
    for q in range(n):
        ax = n - 1 - q
        p1.append(float(np.take(view, 1, axis=ax).sum()))
    proj = [complex(np.vdot(sign_vector(n, k), psi)) for k in range(N_PROJ)]
    return {
        "n": n,
        "idx": [int(i) for i in idx],
        "amps_re": [float(psi[i].real) for i in idx],
        "amps_im": [float(psi[i].imag) for i in idx],
        "p1": p1,
        "proj_re": [p.real for p in proj],
        "proj_im": [p.imag for p in proj],
        "norm2": float(prob.sum()),
    }


def max_error(got: dict, want: dict) -> float:
    """Largest absolute difference over every digest component."""
    assert got["n"] == want["n"] and got["idx"] == want["idx"]
    errs = []
    for key in ("amps_re", "amps_im", "p1", "proj_re", "proj_im"):
        errs.append(np.max(np.abs(np.asarray(got[key]) - np.asarray(want[key]))))
    errs.append(abs(got["norm2"] - want["norm2"]))
    return float(max(errs))
