"""CPU restatement of one rank's share of the column-distributed truncated CPQR
-- TEST INFRASTRUCTURE (see oracle/__init__.py).

Same interface as ``paper_1901_10559_b200.distributed.DeviceCpqrShard`` (the
CUDA kernels of csrc/cpqr_dist.cu), so the host driver and its collectives
(``cpqr_columns_sharded``) run on CPU ranks over gloo.  The arithmetic is
dgeqp3's k-step pivoting rule as the reference reaches it through
scipy.linalg.qr(pivoting=True) (reference linalg.py:97): largest partial
column norm, ties to the lowest position, LAPACK's norm downdate with the
tol3z = sqrt(eps) recompute, Householder vectors with dlarfg's beta/tau.
"""

import numpy as np
import torch

TOL3Z = float(np.sqrt(np.finfo(np.float64).eps))


class OracleCpqrShard:
    def __init__(self, y, col0, k):
        y = y.numpy() if isinstance(y, torch.Tensor) else np.asarray(y)
        self.Y = np.ascontiguousarray(np.asarray(y, dtype=np.float64).T)  # m x n
        self.m, self.n = self.Y.shape
        self.col0, self.k = int(col0), int(k)
        self.vn1 = np.linalg.norm(self.Y, axis=0)
        self.vn2 = self.vn1.copy()
        self.pos = self.col0 + np.arange(self.n, dtype=np.int64)
        self.F = np.zeros((k, self.n))
        self.R = np.zeros((k, self.n))
        self.V = np.zeros((self.m, k))
        self.tau = np.zeros(k)
        self.beta = np.zeros(k)
        self.cand = torch.zeros(4, dtype=torch.float64)
        self.a = torch.zeros(self.m, dtype=torch.float64)
        self._candidate(0)

    def owns(self, col):
        return self.col0 <= col < self.col0 + self.n

    def _candidate(self, pmin):
        val, bpos, col, nxt = -1.0, np.iinfo(np.int64).max, -1, -1
        for j in range(self.n):
            pj = int(self.pos[j])
            if pj == pmin:
                nxt = self.col0 + j
            v = self.vn1[j]
            if pj >= pmin and (v > val or (v == val and pj < bpos)):
                val, bpos, col = v, pj, self.col0 + j
        self.cand[:] = torch.tensor([val, bpos if col >= 0 else -1, col, nxt],
                                    dtype=torch.float64)

    def pivot(self, kk, cs, ps, ck):
        if self.owns(ck) and ck != cs:
            self.pos[ck - self.col0] = ps
        if self.owns(cs):
            c = cs - self.col0
            self.pos[c] = kk
            a = self.Y[:, c] - self.V[:, :kk] @ self.F[:kk, c]
            a[:kk] = 0.0
            self.a[:] = torch.from_numpy(a)
        return self.a

    def step(self, kk, cs, a):
        a = a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        alpha, xnorm = a[kk], np.linalg.norm(a[kk + 1:])
        if xnorm == 0.0:
            tau, beta, scal = 0.0, alpha, 0.0
        else:
            beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            scal = 1.0 / (alpha - beta)
        v = np.zeros(self.m)
        v[kk] = 1.0
        v[kk + 1:] = a[kk + 1:] * scal
        self.V[:, kk] = v
        self.tau[kk], self.beta[kk] = tau, beta
        if self.owns(cs):
            self.R[kk, cs - self.col0] = beta
        z = self.V[:, :kk].T @ v
        act = np.nonzero(self.pos > kk)[0]
        w = self.Y[kk:, act].T @ v[kk:]
        f = tau * (w - self.F[:kk, act].T @ z)
        self.F[kk, act] = f
        rk = self.Y[kk, act] - self.F[:kk, act].T @ self.V[kk, :kk] - f
        self.R[kk, act] = rk
        for i, j in enumerate(act):
            vn1 = self.vn1[j]
            if kk < self.m - 1 and vn1 != 0.0:
                temp = abs(rk[i]) / vn1
                temp = max(0.0, (1.0 + temp) * (1.0 - temp))
                ratio = vn1 / self.vn2[j]
                if temp * ratio * ratio <= TOL3Z:
                    resid = self.Y[kk + 1:, j] - self.V[kk + 1:, :kk + 1] @ self.F[:kk + 1, j]
                    self.vn1[j] = self.vn2[j] = np.linalg.norm(resid)
                else:
                    self.vn1[j] = vn1 * np.sqrt(temp)
        self._candidate(kk + 1)

    def results(self):
        return (torch.from_numpy(self.pos.copy()), torch.from_numpy(self.R.copy()),
                torch.from_numpy(self.beta.copy()))
