"""The native CDF sampler at benchmark sizes (counts pass a
chi-square test against the exact distribution, `tests/conftest.py:154-184`
of the reference): 10^6 shots at n = 20 and 24, and config 3's Sycamore-32
c64 with 10^6 shots, whose 2^32 outcomes are checked through their 16-qubit
marginals (sampling the full state and projecting = sampling the marginal)
against the device's marginal probabilities."""
import numpy as np
import pytest
from scipy import stats

from paper_2512_04216_b200 import _lib, suite
from paper_2512_04216_b200 import statevector as sv

pytestmark = pytest.mark.gpu


def pooled_chisquare(obs: np.ndarray, probs: np.ndarray, shots: int) -> float:
    """One-sample chi-square, bins pooled in ascending-probability order until
    each pool expects >= 5 (the reference helper's pooling, vectorised)."""
    keep = probs > 0
    assert obs[~keep].sum() == 0, "samples on zero-probability outcomes"
    o, e = obs[keep].astype(float), probs[keep] * shots
    order = np.argsort(e, kind="stable")
    o, e = o[order], e[order]
    grp = np.floor(np.cumsum(e) / 5.0).astype(np.int64)
    starts = np.flatnonzero(np.concatenate(([True], grp[1:] != grp[:-1])))
    po, pe = np.add.reduceat(o, starts), np.add.reduceat(e, starts)
    if pe[-1] < 5 and pe.size > 1:  # fold the short tail into its neighbour
        po[-2] += po[-1]
        pe[-2] += pe[-1]
        po, pe = po[:-1], pe[:-1]
    pe *= po.sum() / pe.sum()
    return float(stats.chisquare(po, pe)[1])


@pytest.mark.parametrize("n", [20, 24])
def test_cdf_sampler_chi_square_full_distribution(n):
    shots = 10**6
    c = suite.random_circuit(n, 8 * n, np.random.default_rng(n), measured=False)
    s = sv.DeviceState(n, "c128")
    s.apply_instructions(c.instructions)
    qs = list(range(n))
    probs = s.marginal_probs(qs)
    codes, freq = s.sample_codes(qs, qs, shots, sv.pcg_words(n + 1), _lib.SAMPLER_CDF)
    obs = np.zeros(1 << n, dtype=np.int64)
    obs[codes.astype(np.int64)] = freq.astype(np.int64)
    assert obs.sum() == shots
    assert pooled_chisquare(obs, probs, shots) > 1e-3
    s.close()


def test_sycamore32_million_shots_marginals():
    n, shots = 32, 10**6
    c = suite.sycamore_circuit(4, 8, 20, 0, measured=False)
    s = sv.DeviceState(n, "c64")
    s.apply_instructions(c.instructions)
    qs = list(range(n))
    codes, freq = s.sample_codes(qs, qs, shots, sv.pcg_words(1), _lib.SAMPLER_CDF)
    assert int(freq.sum()) == shots and codes.size > 0.99 * shots  # Porter-Thomas: almost all distinct
    codes = codes.astype(np.uint64)
    for lo in (0, 16):
        marg = s.marginal_probs(list(range(lo, lo + 16)))
        proj = ((codes >> np.uint64(lo)) & np.uint64(0xFFFF)).astype(np.int64)
        obs = np.bincount(proj, weights=freq.astype(np.float64), minlength=1 << 16)
        assert pooled_chisquare(obs, marg, shots) > 1e-3, lo
    s.close()
