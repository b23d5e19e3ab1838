"""Parity rules between the CUDA path and the oracle (readings R17/R18).

* Index sequences: bit-exact. A divergence is *explained* only if the oracle's
  top-2 relative gap at the first divergent step is below ``tau`` (the FP64
  score noise of the explicit-inverse formulation for that input shape, R18);
  otherwise it is a failure. Explained divergences are counted and must stay
  <= ``max_explained`` (fraction) of the locations.
* mean: |dmu| <= 1e-8 * max(|mu_oracle|, std(Z));  s2 and var: |ds2| <= 1e-8 * s2_oracle
  (north_star "1e-8 relative"), checked on every location whose sequence matches.
* flags: EXHAUSTED / SENTINEL bits must agree on matching locations.
"""
from __future__ import annotations

import numpy as np

REL = 1e-8


def tau_for(p: int) -> float:
    # explicit-K^{-1} score noise scale (~2e-5 (2-d), ~4e-5 (3-d grid), ~6e-8 (8-d))
    return 2e-4 if p <= 3 else 1e-6


def compare(gpu: dict, orc: dict, n0: int, zstd: float, tau: float, max_explained: float = 0.01,
            min_explained_allow: int = 1):
    idx_g = np.asarray(gpu["idx"])
    idx_o = np.asarray(orc["idx"])
    M, n = idx_o.shape
    same = (idx_g == idx_o).all(axis=1)
    explained, failures = [], []
    for i in np.where(~same)[0]:
        t = int(np.argmax(idx_g[i] != idx_o[i]))
        if t < n0:
            failures.append((int(i), t, "NN part differs"))
            continue
        gap = orc["gaps"][i, t - n0]
        if gap < max(1e-12, tau):
            explained.append((int(i), t, float(gap)))
        else:
            failures.append((int(i), t, f"oracle gap {gap:.3e} >= tau {tau:.1e}"))
    assert not failures, f"unexplained index divergences: {failures[:10]}"
    allow = max(min_explained_allow, int(max_explained * M))
    assert len(explained) <= allow, f"{len(explained)} explained divergences > {allow}: {explained[:10]}"
    m_g, m_o = np.asarray(gpu["mean"]), orc["mean"]
    s_g, s_o = np.asarray(gpu["s2"]), orc["s2"]
    v_g, v_o = np.asarray(gpu["var"]), orc["var"]
    ok = same
    dm = np.abs(m_g - m_o)[ok]
    lim_m = REL * np.maximum(np.abs(m_o[ok]), zstd)
    assert (dm <= lim_m).all(), f"mean off: max rel {np.max(dm / lim_m) * REL:.3e}"
    ds = np.abs(s_g - s_o)[ok]
    assert (ds <= REL * s_o[ok]).all(), f"s2 off: max rel {np.max(ds / s_o[ok]):.3e}"
    fin = ok & np.isfinite(v_o)
    assert (np.abs(v_g - v_o)[fin] <= REL * v_o[fin]).all()
    assert np.array_equal(np.isnan(v_g[ok]), np.isnan(v_o[ok]))
    fg = np.asarray(gpu["flags"]).astype(np.uint32)
    for bit in (2, 4):  # SENTINEL, EXHAUSTED
        assert np.array_equal(fg[ok] & bit, orc["flags"][ok] & bit), f"flag bit {bit} differs"
    return dict(M=M, identical=int(same.sum()), explained=explained,
                max_rel_mean=float(np.max(dm / np.maximum(np.abs(m_o[ok]), zstd), initial=0.0)),
                max_rel_s2=float(np.max(ds / s_o[ok], initial=0.0)))
