"""Executes the reference-side ctypes binding of INTEGRATION.md verbatim:
the snippets a maintainer of the reference would add, with the reference's
MatVecOperator base stood in by the oracle's (same apply -> _apply counter
protocol), driving the reference algorithm (the oracle restatement of
subspace_iteration_range + direct_svd) with its passes on the GPU."""

import os
import re
import sys
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _snippets():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    return [b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "_lib = C.CDLL" in b
            or "B200DenseOperatorI8" in b]


def test_integration_snippets_run_the_reference_algorithm(monkeypatch):
    from oracle import lowrank_oracle as O
    import paper_0909_4061_b200  # noqa: F401  (builds nothing; the .so is in-tree)
    from paper_0909_4061_b200 import _lib as plib
    lowrank = types.ModuleType("lowrank")
    core = types.ModuleType("lowrank.core")
    core.MatVecOperator = O.Operator
    lowrank.core = core
    monkeypatch.setitem(sys.modules, "lowrank", lowrank)
    monkeypatch.setitem(sys.modules, "lowrank.core", core)
    code = "\n".join(_snippets()).replace('C.CDLL("liblowrank_b200.so")',
                                          f'C.CDLL("{plib.LIB_PATH}")')
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(5)
    A = rng.standard_normal((1500, 700)) * (np.arange(1, 701) ** -0.5)
    ref = O.rsvd(O.Dense(A), 40, 10, 1, 3)
    for cls in ("B200DenseOperator", "B200DenseOperatorI8"):
        op = ns[cls](A)
        basis = O.subspace_iteration_range(op, 50, 1, 3)
        f = O.direct_svd(op, basis.Q)
        assert op.counters.passes == 4     # 3 applications in Alg 4.4 (q = 1) + direct_svd
        assert np.abs(f.sigma - ref[1].sigma).max() <= 1e-10 * ref[1].sigma[0]
