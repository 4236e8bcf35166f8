"""Development repro: the column-slice SpMM against scipy on tiny shapes,
one C-ABI call at a time (synchronizing after each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import torch

from paper_0909_4061_b200 import _lib

g = np.random.default_rng(4)
for (m, n, dens) in [(5, 7, 0.5), (300, 250, 0.04), (3000, 2500, 0.004)]:
    S = sp.random(m, n, density=dens, random_state=4, format="csr")
    rp = torch.from_numpy(S.indptr.astype(np.int64)).cuda()
    ci = torch.from_numpy(S.indices.astype(np.int32)).cuda()
    va = torch.from_numpy(S.data.astype(np.float64)).cuda()
    for ell in (1, 4, 5, 8, 48):
        X = torch.from_numpy(g.standard_normal((n, ell))).cuda()
        Y = torch.zeros((m, ell), dtype=torch.float64, device="cuda")
        print("ptrs mod 16:", rp.data_ptr() % 16, ci.data_ptr() % 16, va.data_ptr() % 16,
              X.data_ptr() % 16, Y.data_ptr() % 16, flush=True)
        try:
            _lib.call("lr_csr_spmm", _lib.handle(0), _lib.F64, m, n, ell, _lib.ptr(rp),
                      _lib.ptr(ci), _lib.ptr(va), _lib.ptr(X), _lib.ld(X), _lib.ptr(Y),
                      _lib.ld(Y), 0)
            torch.cuda.synchronize()
            print(m, n, ell, np.abs(Y.cpu().numpy() - S @ X.cpu().numpy()).max(), flush=True)
        except Exception as e:
            print("ERR", m, n, ell, e, flush=True)
            sys.exit(1)
