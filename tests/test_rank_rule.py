"""rs_rank_rule (host C) against rankred.rank_rule_fast (Python) -- the eps-rank
rule of rankred.py:129-148 on top-b Ritz values; runs without a GPU."""
import ctypes

import numpy as np
import pytest

from paper_1606_09218_b200 import _native as nat
from paper_1606_09218_b200.rankred import rank_rule_fast


def _c_rule(thetas, traces, b, n, eps, forced, limit, iters):
    m = len(traces)
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    tr = np.ascontiguousarray(traces, dtype=np.float64)
    ro, to, so = (ctypes.c_int64 * m)(), (ctypes.c_double * m)(), (ctypes.c_double * m)()
    fo = None
    if forced is not None:
        fo = (ctypes.c_int64 * m)(*[int(f) if f is not None else 0 for f in forced])
    rc = nat.lib().rs_rank_rule(th.ctypes.data, tr.ctypes.data, m, b, n, eps,
                                ctypes.addressof(fo) if fo is not None else None,
                                limit if limit is not None else 0, iters, ctypes.addressof(ro),
                                ctypes.addressof(to), ctypes.addressof(so))
    assert rc == 0
    return [(ro[l] if ro[l] > 0 else None, to[l], so[l]) for l in range(m)]


@pytest.mark.parametrize("b", [16, 24, 64, 192])
@pytest.mark.parametrize("seed", range(6))
def test_rank_rule_matches_python(b, seed):
    rng = np.random.default_rng(seed)
    n = 256 if b < 192 else 2048
    decay = rng.uniform(0.3, 1.2)
    th = np.stack([np.sort(rng.uniform(0.5, 1.0, b) * np.exp(-decay * np.arange(b)))[::-1]
                   * 10.0 ** rng.uniform(-3, 6) for _ in range(3)])
    if seed % 3 == 0:
        th[1, -3:] = -1e-18          # clipped negatives
    traces = th.clip(0).sum(1) * (1 + rng.uniform(0, 1e-12, 3))
    for eps in (1e-6, 1e-8, 1e-12):
        for forced in (None, (3, 5, 7)):
            for limit in (None, 4):
                want = rank_rule_fast(th.reshape(-1).tolist(), traces.tolist(), n, eps, forced,
                                      limit, 2)
                got = _c_rule(th.reshape(-1), traces, b, n, eps, forced, limit, 2)
                for (rw, tw, sw), (rg, tg, sg) in zip(want, got):
                    assert rw == rg
                    assert sg == sw          # same summation order: bit-identical
                    if rw is not None:
                        assert tg == tw


def test_rank_rule_zero_spectrum():
    got = _c_rule(np.zeros(3 * 16), np.zeros(3), 16, 256, 1e-6, None, None, 2)
    want = rank_rule_fast([0.0] * 48, [0.0] * 3, 256, 1e-6, None, None, 2)
    assert [g[0] for g in got] == [w[0] for w in want]
