import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1901_10559_b200 as ids
for (m, n), k in [((100, 2000), 20), ((40, 1000), 10), ((60, 60), 5), ((60, 60), 60)]:
    rng = np.random.default_rng(m + n)
    base = rng.standard_normal((m, k)) @ rng.standard_normal((k, n))
    y = base + 1e-3 * rng.standard_normal((m, n))
    f = ids.cpqr(y, k)
    w = oracle.cpqr(y, k)
    qq = np.abs(f.q.T @ f.q - np.eye(k)).max()
    sq = np.sign(np.sum(f.q * w.q, axis=0))
    dq = np.abs(f.q - w.q * sq).max()
    r_sel = np.abs(f.r[:, :k] - (w.r[:, :k] * sq[:, None])).max()
    # compare trailing columns by column id
    pos_o = {c: i for i, c in enumerate(w.perm)}
    tr = [pos_o[c] for c in f.perm[k:]]
    r_tr = np.abs(f.r[:, k:] - (w.r[:, tr] * sq[:, None])).max()
    err = np.linalg.norm(f.q @ f.r - y[:, f.perm]) / np.linalg.norm(y)
    qr_sel = np.abs(f.q @ f.r[:, :k] - y[:, f.perm[:k]]).max()
    print((m, n, k), f"QtQ-I {qq:.2e} dQ {dq:.2e} dR_sel {r_sel:.2e} dR_tr {r_tr:.2e} err {err:.2e} qr_sel {qr_sel:.2e}", flush=True)
