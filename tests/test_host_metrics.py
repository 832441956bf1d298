"""Header-only host API: the correlation metrics (include/gsr/metrics.hpp,
SPEC.md:534-563) against scipy and an O(m²) tau-b pair count, and the worker
pool (include/gsr/threads.hpp, reference proj/include/gsr/threads.hpp:17-52)
for bit-identical results across worker counts."""
import itertools
import os
import subprocess

import numpy as np
import pytest
from scipy import stats

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def drv(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("host") / "host_check")
    subprocess.run(["g++", "-O2", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-pthread", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_check.cpp"), "-o", exe], check=True)
    return exe


def _metrics(drv, a, b):
    inp = f"{len(a)}\n" + " ".join(repr(float(x)) for x in a) + "\n" + " ".join(repr(float(x)) for x in b) + "\n"
    out = subprocess.run([drv, "metrics"], input=inp, capture_output=True, text=True, check=True).stdout.split()
    if out[0] == "ShapeError":
        raise ValueError(" ".join(out))
    return [float(x) for x in out]


def _kendall_pairs(a, b):
    """tau-b by the O(m²) pair count"""
    nc = nd = ta = tb = 0
    for i, j in itertools.combinations(range(len(a)), 2):
        da, db = np.sign(a[i] - a[j]), np.sign(b[i] - b[j])
        if da == 0 and db == 0:
            continue
        if da == 0:
            ta += 1
        elif db == 0:
            tb += 1
        elif da == db:
            nc += 1
        else:
            nd += 1
    return (nc - nd) / np.sqrt((nc + nd + ta) * (nc + nd + tb))


@pytest.mark.parametrize("seed", range(6))
def test_metrics_match_scipy_and_pair_count(drv, seed):
    rng = np.random.default_rng(seed)
    m = 50
    a = rng.integers(0, 6, m).astype(float) if seed % 2 else rng.normal(size=m)   # heavy ties on odd seeds
    b = np.round(a + rng.normal(scale=1.5, size=m), 0 if seed % 3 == 0 else 6)
    p, s, k, r2 = _metrics(drv, a, b)
    assert abs(p - stats.pearsonr(a, b)[0]) <= 1e-12
    assert abs(s - stats.spearmanr(a, b)[0]) <= 1e-12
    assert abs(k - stats.kendalltau(a, b)[0]) <= 1e-12          # scipy's default is tau-b
    assert abs(k - _kendall_pairs(a, b)) <= 1e-12
    assert abs(r2 - (1 - ((b - a) ** 2).sum() / ((b - b.mean()) ** 2).sum())) <= 1e-12


def test_metrics_known_answers_and_markers(drv):
    a = np.arange(10, dtype=float)
    assert _metrics(drv, a, a) == [1.0, 1.0, 1.0, 1.0]
    p, s, k, _ = _metrics(drv, a, -a)
    assert (p, s, k) == (-1.0, -1.0, -1.0)
    p, s, k, _ = _metrics(drv, a, np.exp(a))                     # monotone transform: rank metrics stay 1
    assert s == 1.0 and k == 1.0 and p < 1.0
    assert _metrics(drv, np.full(10, a.mean()), a)[3] == 0.0     # pred = mean(truth) → R² = 0
    out = _metrics(drv, a, np.full(10, 3.0))                      # constant input → explicit NaN marker
    assert all(np.isnan(out))
    with pytest.raises(ValueError, match="ShapeError"):
        _metrics(drv, a[:1], a[:1])


def test_kendall_adjacent_swap(drv):
    """swapping one adjacent pair of distinct values changes tau by 2/C(m,2)"""
    a = np.arange(20, dtype=float)
    b = a.copy()
    b[[7, 8]] = b[[8, 7]]
    k = _metrics(drv, a, b)[2]
    assert abs(k - (1 - 2 * 2 / (20 * 19))) <= 1e-15


@pytest.mark.parametrize("n", [1, 7, 1000, 100_003])
def test_thread_pool_bit_identical_across_worker_counts(drv, n):
    outs = set()
    for t in (1, 2, 3, 8, 16):
        r = subprocess.run([drv, "threads", str(t), str(n)], capture_output=True, text=True, check=True).stdout.split()
        assert int(r[0]) == t and r[2] == "1"
        outs.add(r[1])
    assert len(outs) == 1
