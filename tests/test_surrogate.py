"""The search's cost model (NEXT-3, P:369 step 3 / P:371-377): graph features and the
gradient-boosted regression-tree ensemble, host-only (runs without a GPU).

Pins: hand-derived feature vectors; scikit-learn's GradientBoostingRegressor with the same
hyper-parameters (squared loss, mean init, 60 rounds, depth 3, shrinkage 0.2, min 2 samples
per leaf, exact splits) as an independent implementation of the same algorithm; exact
recovery of a step function; generalisation on an additive target."""
import math

import numpy as np
import pytest

asp = pytest.importorskip("paper_2212_10432_b200")

N_OPS, N_PAR = 24, 17  # parameter classes incl. SET_RESOURCE xcache and stream (R-conc)


def test_feature_layout_hand_derived():
    f = asp.Graph("COMPRESS; BMT_NNZ_BLOCK(8); THREAD_BITMAP_RED_G; GMEM_ATOM_RED").features()
    assert f.shape == (N_OPS + N_PAR + 1,)
    exp = np.zeros_like(f)
    exp[7] = 1    # COMPRESS
    exp[13] = 1   # BMT_NNZ_BLOCK
    exp[17] = 1   # THREAD_BITMAP_RED_G
    exp[N_OPS + 1] = math.log2(9)   # BMT_NNZ_BLOCK nnz = 8
    exp[-1] = 1   # one leaf
    assert np.array_equal(f, exp)


def test_feature_branches_and_means():
    g = asp.Graph("BIN(t=[4,64]) { COMPRESS; BMT_ROW_BLOCK(1); THREAD_TOTAL_RED; SET_RESOURCE(tpb=128); GMEM_ATOM_RED"
                  " | COMPRESS; BMW_ROW_BLOCK(1); WARP_TOTAL_RED; SET_RESOURCE(tpb=512); GMEM_ATOM_RED"
                  " | COMPRESS; BMTB_ROW_BLOCK(1); SHMEM_TOTAL_RED; GMEM_ATOM_RED }")
    f = g.features()
    assert f[4] == 1 and f[7] == 3 and f[23] == 2          # BIN, 3 x COMPRESS, 2 x SET_RESOURCE
    assert f[10] == 1 and f[9] == 1 and f[8] == 1          # BMT/BMW/BMTB_ROW_BLOCK
    assert f[N_OPS + 6] == pytest.approx((math.log2(129) + math.log2(513)) / 2)   # mean tpb class
    assert f[-1] == 3


def test_feature_stream_class():
    """R-conc: SET_RESOURCE stream is its own parameter class (index 10, after xcache)."""
    f = asp.Graph("DIA_DECOM(0.5) { DIA; SET_RESOURCE(stream=1) | COMPRESS; BMT_NNZ_BLOCK(4); "
                  "THREAD_BITMAP_RED_G; GMEM_ATOM_RED }").features()
    assert f[N_OPS + 10] == pytest.approx(1.0)   # mean log2(1 + 1) over the one SET_RESOURCE


def _gbr_sklearn(X, y, Xq):
    ens = pytest.importorskip("sklearn.ensemble")
    m = ens.GradientBoostingRegressor(loss="squared_error", learning_rate=0.2, n_estimators=60, max_depth=3,
                                      min_samples_leaf=2, min_samples_split=4, subsample=1.0,
                                      max_features=None, random_state=0)
    m.fit(X, y)
    return m.predict(Xq)


@pytest.mark.parametrize("seed", range(4))
def test_matches_sklearn_gbr(seed):
    """Same algorithm, independent implementation.  With several features, equal-gain splits
    on different features (common in small nodes) are broken differently (sklearn visits
    features in a random order), which changes predictions between training points but not
    at them: compare on the training points.  With one feature there are no such ties:
    compare on fresh query points too (thresholds = midpoints)."""
    g = np.random.default_rng(seed)
    n, d = 40, 6
    X = g.uniform(-1, 1, (n, d)).astype(np.float32).astype(np.float64)  # sklearn trees split in fp32
    y = np.sin(3 * X[:, 0]) + X[:, 1] * X[:, 2] + 0.1 * g.normal(size=n)
    np.testing.assert_allclose(asp.surrogate_fit_predict(X, y, X), _gbr_sklearn(X, y, X), rtol=0, atol=1e-9)
    x1 = X[:, :1]
    q1 = g.uniform(-1, 1, (25, 1)).astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(asp.surrogate_fit_predict(x1, y, q1), _gbr_sklearn(x1, y, q1), rtol=0, atol=1e-9)


def test_step_function_exact():
    X = np.array([[0.1 * i, 0.0] for i in range(20)])
    y = np.where(X[:, 0] > 0.95, 3.0, 1.0)
    p = asp.surrogate_fit_predict(X, y, np.array([[0.2, 0.0], [1.7, 0.0]]))
    np.testing.assert_allclose(p, [1.0, 3.0], atol=1e-4)   # residual shrinks as 0.8^60


def test_generalises_additive():
    g = np.random.default_rng(7)
    X = g.uniform(0, 4, (120, 5))
    y = X[:, 0] + 2 * np.floor(X[:, 1])
    Xq = g.uniform(0, 4, (200, 5))
    yq = Xq[:, 0] + 2 * np.floor(Xq[:, 1])
    p = asp.surrogate_fit_predict(X, y, Xq)
    assert np.mean(np.abs(p - yq)) < 0.25 * np.mean(np.abs(yq - y.mean()))


def test_degenerate_and_deterministic():
    Xq = np.zeros((3, 2))
    assert np.array_equal(asp.surrogate_fit_predict(np.zeros((0, 2)), np.zeros(0), Xq), np.zeros(3))
    assert np.array_equal(asp.surrogate_fit_predict(np.ones((1, 2)), np.array([5.0]), Xq), np.full(3, 5.0))
    g = np.random.default_rng(1)
    X, y = g.normal(size=(30, 4)), g.normal(size=30)
    a = asp.surrogate_fit_predict(X, y, X)
    b = asp.surrogate_fit_predict(X, y, X)
    assert np.array_equal(a, b)
