"""CPU oracle for the error metrics -- TEST INFRASTRUCTURE (see oracle/__init__.py).

Restates, from the reference's behaviour:
* ``derive_seed`` (reference ``pkg/src/idsketch/bench.py:116-120``): first
  32-bit word of ``SeedSequence([master, *tags])``;
* ``est_spectral_norm`` (``estimators.py:26-88``): adjoint consistency probe,
  then ``iters`` steps of normalized power iteration on B'B from ``probes``
  Gaussian starts; the value is max ||B v|| / ||v|| over the final iterates.
  Random draws in the reference's order: x (cols), y (len(Bx)), starts
  (probes x cols), all from ``default_rng(seed)``;
* ``id_residual_operator`` (``estimators.py:91-110``): x -> A[:, J](P x) - A x
  and y -> P'(A[:, J]' y) - A' y;
* ``matrix_operator`` (``estimators.py:113-121``).
"""

import numpy as np

ADJOINT_RTOL = 1e-10  # estimators.py:14


def derive_seed(master, *tags):
    words = np.random.SeedSequence([int(master)] + [int(t) for t in tags]).generate_state(1)
    return int(words[0])


def est_spectral_norm(apply, apply_adjoint, cols, iters=10, probes=2, seed=None):
    if cols < 1:
        raise ValueError("cols must be positive")
    if iters < 0 or probes < 1:
        raise ValueError("need iters >= 0 and probes >= 1")
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(cols)
    bx = np.asarray(apply(x), dtype=np.float64)
    y = rng.standard_normal(bx.shape[0])
    bty = np.asarray(apply_adjoint(y), dtype=np.float64)
    nrm = np.linalg.norm
    scale = nrm(bx) * nrm(y) + nrm(x) * nrm(bty)
    if abs(float(bx @ y) - float(x @ bty)) > ADJOINT_RTOL * max(scale, 1.0):
        raise ValueError("operator pair failed the adjoint test")
    starts = rng.standard_normal((probes, cols))
    best = 0.0
    for v in starts:
        n0 = nrm(v)
        if n0 == 0.0:
            continue
        v = v / n0
        for _ in range(iters):
            v = np.asarray(apply_adjoint(np.asarray(apply(v), dtype=np.float64)), dtype=np.float64)
            nv = nrm(v)
            if nv == 0.0:
                break
            v = v / nv
        if nrm(v) == 0.0:
            continue
        best = max(best, float(nrm(apply(v)) / nrm(v)))
    return best


def id_residual_operator(a, cols, coeffs):
    sel = a[:, cols]

    def apply(x):
        return np.asarray(sel @ (coeffs @ x) - a @ x).ravel()

    def apply_adjoint(y):
        return np.asarray(coeffs.T @ (sel.T @ y) - a.T @ y).ravel()

    return apply, apply_adjoint


def matrix_operator(a):
    return (lambda x: np.asarray(a @ x).ravel()), (lambda y: np.asarray(a.T @ y).ravel())
