"""k-fold cross-validation along the λ path on the GPU (reading R35)
against the oracle's cv_path (itself pinned to scikit-learn): the held-out residual hook, then the
whole CV curve and the selected index."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import cuda_ok

pytestmark = pytest.mark.gpu

if cuda_ok():
    import torch
    from paper_2006_03970_b200 import Problem
    from paper_2006_03970_b200.path import cv_path


def test_residual_hook():
    cfg = synth.scaled(synth.CONFIGS["cfg3"], n=5000)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    rng = np.random.default_rng(0)
    with Problem(A, b) as P:
        for nnz in (0, 1, 37, 4999):
            x = np.zeros(cfg.n)
            idx = rng.choice(cfg.n, nnz, replace=False)
            x[idx] = rng.standard_normal(nnz)
            ref = float(np.sum((A.T @ x - b) ** 2))
            assert P.residual(x) == pytest.approx(ref, rel=1e-12)
            dx = torch.from_numpy(x).cuda()
            assert P.residual_device(dx.data_ptr()) == pytest.approx(ref, rel=1e-12)


@pytest.mark.parametrize("name,n,k", [("cfg2", 20_000, 5), ("cfg1", None, 4)])
def test_cv_path_matches_oracle(name, n, k):
    cfg = synth.CONFIGS[name] if n is None else synth.scaled(synth.CONFIGS[name], n=n)
    A = synth.design(cfg)
    b, _ = synth.response(cfg)
    cs = [0.9, 0.6, 0.4, 0.25, 0.15]
    lm = float(np.max(np.abs(oracle.aty(A, b))))
    dA = torch.from_numpy(A).cuda()  # (n, m): column-major m × n
    st = torch.cuda.current_stream()

    def make(rows):
        sub = dA[:, torch.from_numpy(rows).cuda()].contiguous()
        bs = torch.from_numpy(np.ascontiguousarray(b[rows])).cuda()
        return Problem.from_device(sub.data_ptr(), bs.data_ptr(), len(rows), cfg.n, st.cuda_stream, keep=(sub, bs))

    cv_g, best_g = cv_path(make, cfg.m, cfg.alpha, cs, lm, k=k, tol=1e-9)
    cv_c, best_c = oracle.cv_path(A, b, cfg.alpha, cs, k=k, tol=1e-9)
    np.testing.assert_allclose(cv_g, cv_c, rtol=1e-7)
    assert best_g == best_c
