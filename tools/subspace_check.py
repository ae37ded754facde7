import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import qdwh_oracle as O
from paper_2104_14186_b200 import matgen, qdwh
for n, k, fam, seed in [(2048, 20, 'logsigned', 7), (4096, 41, 'logsigned', 42), (3072, 31, 'logsigned', 1), (2048, 60, 'uniform', 3), (4096, 200, 'uniform', 5)]:
    lam = matgen.config_eigenvalues(fam, n, seed)
    q, _ = np.linalg.qr(O.gaussian_matrix(n, n, seed))
    a = (q * lam) @ q.T; a = 0.5 * (a + a.T)
    c = matgen.largest_k_shift(lam, k)
    r = qdwh.partial_eig_request(a, 'largest', c, k)
    st = r.stage_seconds if hasattr(r, 'stage_seconds') else None
    v = np.asarray(r.v)
    res = np.linalg.norm(a @ v - v * r.lambda_minus) / np.linalg.norm(a)
    print(n, k, fam, r.count(), r.subspace_size, '%.1e' % res, [round(x*1e3,2) for x in st][:4] if st else '')
