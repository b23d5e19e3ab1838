"""GPU parity for row f3 (separable lengthscales; reading R23):
laGP_alc_batch_sep through the C ABI against oracle.alc_batch_sep on seeded
inputs, every formulation, with the parity rules of tests/parity.py (bit-exact
index sequences up to explained near ties; mean/s2/var within 1e-8)."""
import numpy as np
import pytest

import oracle
from lagp_data import make_config
from parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    return torch, torch.device("cuda", 0)


@pytest.fixture(scope="module")
def lagp():
    import paper_1310_5182_b200 as m

    m.lib()
    return m


def T(torch, dev, a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


CASES = [
    ("C1", 64, None, [0.02, 0.09], {}),  # 2-d, anisotropic
    ("C2", 48, 20000, [0.3, 0.5, 0.9, 2.0, 0.4, 1.5, 0.7, 5.0], {}),  # 8-d borehole, mixed relevance
    ("C3", 48, None, [0.05, 0.4, 3.0], {}),  # LGBB grid: weighted-distance ties at the N'-th NN
    ("C1", 9, 3000, [0.5, 0.01], dict(n0=4, n=128, Nprime=300)),  # n = LAGP_NMAX
]


@pytest.mark.parametrize("name,M,N,theta,over", CASES)
@pytest.mark.parametrize("form", ["explicit", "explicit_dfma", "incremental"])
def test_alc_batch_sep_vs_oracle(torch_dev, lagp, name, M, N, theta, over, form):
    torch, dev = torch_dev
    cfg = make_config(name, M=M, N=N, **over)
    X, Z, XX = cfg["X"], cfg["Z"], cfg["XX"]
    r = lagp.alc_batch_sep(T(torch, dev, X), T(torch, dev, Z), T(torch, dev, XX), theta, cfg["g"], cfg["n0"],
                           cfg["n"], cfg["Nprime"], form=form, gaps=True)
    g = {k: v.cpu().numpy() for k, v in r.items() if hasattr(v, "cpu")}
    o = oracle.alc_batch_sep(X, Z, XX, theta, cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    # R18 on the rescaled inputs the oracle ran on (isotropic with d = 1, reading R23)
    scaled = dict(cfg, X=oracle.sep_scale(X, theta), XX=oracle.sep_scale(XX, theta), d=1.0)
    rep = check(g, o, scaled, form, label=f"sep-{name}")
    print(name, form, rep)

