"""Model-Driven Format Compression (NEXT-2, §V-D): the oracle's array-model fitter
pinned by SPEC's examples and by exhaustive soundness, the C-ABI fitter bit-exact against
the oracle on structured and random arrays (host only), and -- on the GPU -- plans whose
first-row / origin-row arrays are replaced by models computing the same y."""
import os

import numpy as np
import pytest

import synth
from oracle import model_ref as M
from oracle import spmv as S

asp = pytest.importorskip("paper_2212_10432_b200")


# ------------------------------------------------------------------ oracle pins
def test_spec_examples():
    # S:338 "[0,64,128,192] -> linear(k=64,b=0), 0 patches" ("row_offset=64*bid")
    assert M.fit_array_model([0, 64, 128, 192]) == (M.LINEAR, 0, 64, 0, 1, [])
    # S:339 "[0,64,999,192] -> linear(k=64,b=0) with patch {2:999}"
    assert M.fit_array_model([0, 64, 999, 192]) == (M.LINEAR, 0, 64, 0, 1, [(2, 999)])
    # S:340 "cryptographic-random 64-entry array -> none"
    r = np.random.default_rng(1).integers(0, 2**40, 64)
    assert M.fit_array_model(r) is None


def test_hypotheses_closed_forms():
    i = np.arange(1000)
    assert M.fit_array_model(7 + 3 * i) == (M.LINEAR, 7, 3, 0, 1, [])
    per = 5 + 100 * (i // 32) + 2 * (i % 32)                 # periodic linear, period 32
    assert M.fit_array_model(per) == (M.PERIODIC, 5, 100, 2, 32, [])
    step = 4 + 9 * (i // 3)                                    # step, run length 3 (not a power of 2)
    assert M.fit_array_model(step) == (M.STEP, 4, 9, 0, 3, [])
    const = np.full(10, 6)                                     # constant = linear with k = 0
    assert M.fit_array_model(const) == (M.LINEAR, 6, 0, 0, 1, [])


def test_patch_budget_boundary():
    a = list(range(0, 200, 2))
    for j in range(8):
        a[10 * j + 5] = -1
    m = M.fit_array_model(a)
    assert m[:5] == (M.LINEAR, 0, 2, 0, 1) and len(m[5]) == 8
    a[95] = -1                                                 # a 9th error
    assert M.fit_array_model(a) is None
    assert M.fit_array_model(a, budget=9)[:2] == (M.LINEAR, 0)


@pytest.mark.parametrize("seed", range(20))
def test_soundness_exhaustive(seed):
    """S:353 'for every array and fitted model, forall i: model_with_patches(i) == array[i]'."""
    g = np.random.default_rng(seed)
    n = int(g.integers(2, 600))
    i = np.arange(n)
    kind = seed % 4
    if kind == 0:
        a = int(g.integers(-50, 50)) + int(g.integers(-9, 9)) * i
    elif kind == 1:
        w = int(2 ** g.integers(1, 8))
        a = int(g.integers(0, 9)) + int(g.integers(0, 99)) * (i // w) + int(g.integers(0, 5)) * (i % w)
    elif kind == 2:
        w = int(g.integers(1, 40))
        a = int(g.integers(0, 9)) + int(g.integers(1, 9)) * (i // w)
    else:
        a = np.cumsum(g.integers(0, 7, n))
    a = np.array(a, np.int64)
    for j in g.integers(0, n, int(g.integers(0, 4))):
        a[j] += int(g.integers(1, 1000))
    m = M.fit_array_model(a)
    if m is not None:
        assert [M.evaluate(m, j) for j in range(n)] == a.tolist()


# ------------------------------------------------------------------ C-ABI fitter vs oracle
def _cases():
    g = np.random.default_rng(11)
    out = [np.array([0, 64, 128, 192]), np.array([0, 64, 999, 192]), np.array([3, 3]), np.array([5, 1]),
           np.arange(1000) * 7 + 2, 5 + 100 * (np.arange(700) // 32) + 2 * (np.arange(700) % 32),
           4 + 9 * (np.arange(50) // 3), g.integers(0, 2**40, 64), np.cumsum(g.integers(0, 3, 300))]
    for s in range(40):
        n = int(g.integers(2, 400))
        i = np.arange(n)
        w = int(2 ** g.integers(1, 6))
        a = [i * int(g.integers(-5, 6)), (i // w) * 17 + (i % w) * 3, (i // int(g.integers(1, 9))) * 4][s % 3]
        a = np.array(a, np.int64) + int(g.integers(-100, 100))
        for j in g.integers(0, n, int(g.integers(0, 11))):
            a[j] = int(g.integers(-10**6, 10**6))
        out.append(a)
    return out


@pytest.mark.parametrize("k", range(49))
def test_abi_matches_oracle(k):
    a = _cases()[k]
    for budget in (0, 3, 8):
        ref = M.fit_array_model(a, budget)
        got = asp.fit_array_model(a, budget)
        assert got == ref, (k, budget, got, ref)


def _long_cases():
    """Arrays above 8192 entries, where the C-ABI (as the device build) first probes the
    first 4096 entries and the mid / last pairs (model_may_fit) before reading the rest:
    patches beyond the prefix, near the middle and at the end; a step longer than the probe;
    periodic; random and cumulative arrays."""
    g = np.random.default_rng(23)
    out = []
    for n in (9000, 20000, 33000):
        i = np.arange(n, dtype=np.int64)
        lin = 11 + 4 * i
        for pos in ([5000], [n // 2], [n // 2 + 1], [n - 1], [n - 2], [100, 7000, n - 1], list(range(4090, 4099))):
            a = lin.copy()
            for j in pos:
                a[j] += 7
            out.append(a)
        out.append(3 + 6 * (i // 5000))        # step wider than the probe
        out.append(3 + 6 * (i // 700))         # step inside the probe
        out.append(5 + 100 * (i // 64) + 2 * (i % 64))
        out.append(g.integers(0, 2**31, n))
        out.append(np.cumsum(g.integers(0, 3, n)))
    return out


@pytest.mark.parametrize("k", range(36))
def test_abi_matches_oracle_long(k):
    a = _long_cases()[k]
    for budget in (0, 3, 8):
        assert asp.fit_array_model(a, budget) == M.fit_array_model(a, budget), (k, budget)


# ------------------------------------------------------------------ GPU: compressed plans
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _uniform_rows(m, n, L, seed):
    g = np.random.default_rng(seed)
    rows = np.repeat(np.arange(m), L)
    cols = np.concatenate([np.sort(g.choice(n, L, replace=False)) for _ in range(m)])
    return synth.Coo(m, n, rows.astype(np.int64), cols.astype(np.int64), g.integers(-4, 5, m * L).astype(np.float64))


def _alternating(m, n, seed):
    g = np.random.default_rng(seed)
    rows, cols = [], []
    for r in range(m):
        L = 2 if r % 2 == 0 else 7
        rows.append(np.full(L, r))
        cols.append(np.sort(g.choice(n, L, replace=False)))
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    return synth.Coo(m, n, rows.astype(np.int64), cols.astype(np.int64),
                     g.integers(-4, 5, rows.shape[0]).astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("case,graph,min_models", [
    ("uniform", "COMPRESS; BMT_NNZ_BLOCK(16); THREAD_BITMAP_RED_G; GMEM_ATOM_RED", 1),           # first_row = 2t
    ("uniform", "COMPRESS; BMT_NNZ_BLOCK(16); BMT_PAD(GLOBAL,2); THREAD_BITMAP_RED_G; GMEM_ATOM_RED", 1),
    ("uniform", "COMPRESS; BMW_NNZ_BLOCK(256); BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; WARP_SEG_ADD_RED; "
                "GMEM_ATOM_RED", 1),
    ("alternating", "BIN(t=[4]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; GMEM_ATOM_RED }", 2),  # origin = 2r(+1)
    ("alternating", "BIN(t=[4]) { COMPRESS; BMT_NNZ_BLOCK(14); THREAD_BITMAP_RED_G; GMEM_ATOM_RED }", 3),
])
@pytest.mark.parametrize("beta", [0.0, 2.0])
def test_gpu_compressed_plans(case, graph, min_models, beta):
    torch = _gpu()
    coo = _uniform_rows(3000, 2500, 8, 2) if case == "uniform" else _alternating(4000, 3000, 3)
    A = asp.Matrix.from_coo(coo.m, coo.n, coo.row, coo.col, coo.val)
    x, y0 = synth.vectors(coo.n, coo.m, 4, np.float64, True)
    yref, _ = S.spmv_coo(coo.m, coo.row, coo.col, coo.val, x, 1.0, beta, y0)
    outs = []
    for mdc in (True, False):
        if mdc:
            os.environ.pop("AS_NO_MDC", None)
        else:
            os.environ["AS_NO_MDC"] = "1"
        try:
            P = asp.Plan(A, graph, device=0)
        finally:
            os.environ.pop("AS_NO_MDC", None)
        info = P.info()
        assert (info["modeled_arrays"] >= min_models) if mdc else info["modeled_arrays"] == 0
        dy = torch.from_numpy(y0.copy()).cuda()
        P.spmv(1.0, torch.from_numpy(x).cuda(), beta, dy)
        torch.cuda.synchronize()
        outs.append((dy.cpu().numpy(), info["bytes_model"]))
    assert np.array_equal(outs[0][0], yref) and np.array_equal(outs[1][0], yref)
    assert outs[0][1] < outs[1][1]  # the modeled arrays left the bytes model
