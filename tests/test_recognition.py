"""Recognition path: projection, explained variance,
k-NN and dense PCA.  The oracle (oracle/recognition.py) is pinned to
tests/golden/recog.json (produced by running the reference,
tests/golden/make_golden_recog.py); the device path is checked against both
(reference tests/test_pca.py and tests/test_datasets.py knn cases are the
model)."""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from recipes import knn_case, recog_samples, sparse_loadings  # noqa: E402

from oracle import recognition as orc  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "recog.json")))


def _case_inputs(c):
    S = recog_samples(c["seed"], c["n"], c["f"])
    L = sparse_loadings(c["loading_seed"], c["f"], c["m"] + 1, max(2, c["f"] // 5))
    return S, L


# ------------------------------------------------------------------ oracle


@pytest.mark.parametrize("c", GOLD["projection"], ids=lambda c: f"n{c['n']}f{c['f']}")
def test_oracle_projection_matches_reference(c):
    S, L = _case_inputs(c)
    comps, sv, mu = orc.dense_pca(S, c["m"])
    np.testing.assert_allclose(comps, c["pca_components"], atol=1e-10)
    np.testing.assert_allclose(sv, c["pca_singular_values"], rtol=1e-12)
    np.testing.assert_allclose(mu, c["pca_mean"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(orc.embed(S, comps), c["project_pca"], atol=1e-10)
    np.testing.assert_allclose(orc.embed(S, L), c["project_sparse"], rtol=1e-12, atol=1e-12)
    mean_given = S[: c["n"] // 2].mean(axis=0)
    np.testing.assert_allclose(orc.embed(S, L, mean_given), c["project_sparse_given_mean"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(orc.variance_explained(S, comps), c["ev_pca"], rtol=1e-10)
    np.testing.assert_allclose(orc.variance_explained(S, L), c["ev_sparse"], rtol=1e-10, atol=1e-14)
    assert c["ev_sparse"][-1] == 0.0  # zero component credited nothing


@pytest.mark.parametrize("c", GOLD["knn"], ids=lambda c: f"r{c['r']}t{c['t']}")
def test_oracle_knn_matches_reference(c):
    train, labels, test = knn_case(c["seed"], c["r"], c["t"], c["dim"], c["n_labels"], c["dup"])
    for k, pred in c["pred"].items():
        np.testing.assert_array_equal(orc.knn_predict(train, labels, test, int(k)), pred)


# ------------------------------------------------------------------ device

gps = None


def _gps():
    global gps
    if gps is None:
        import paper_1312_6182_b200 as g

        gps = g
    return gps


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLD["projection"], ids=lambda c: f"n{c['n']}f{c['f']}")
def test_device_projection_and_variance_vs_reference(c):
    g = _gps()
    S, L = _case_inputs(c)
    comps = np.asarray(c["pca_components"])
    np.testing.assert_allclose(g.project(S, comps), c["project_pca"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(g.project(S, L), c["project_sparse"], rtol=1e-10, atol=1e-11)
    mean_given = S[: c["n"] // 2].mean(axis=0)
    np.testing.assert_allclose(g.project(S, L, mean=mean_given), c["project_sparse_given_mean"], rtol=1e-10,
                               atol=1e-11)
    np.testing.assert_allclose(g.explained_variance(S, comps), c["ev_pca"], rtol=1e-10)
    np.testing.assert_allclose(g.explained_variance(S, L), c["ev_sparse"], rtol=1e-10, atol=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLD["projection"], ids=lambda c: f"n{c['n']}f{c['f']}")
def test_device_pca_fit_vs_reference(c):
    g = _gps()
    S, _ = _case_inputs(c)
    model = g.pca_fit(S, c["m"])
    np.testing.assert_allclose(model.singular_values, c["pca_singular_values"], rtol=1e-10)
    np.testing.assert_allclose(model.components, c["pca_components"], atol=1e-8)
    np.testing.assert_allclose(model.mean, c["pca_mean"], rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLD["knn"], ids=lambda c: f"r{c['r']}t{c['t']}")
def test_device_knn_vs_reference(c):
    g = _gps()
    train, labels, test = knn_case(c["seed"], c["r"], c["t"], c["dim"], c["n_labels"], c["dup"])
    for k, pred in c["pred"].items():
        got, acc = g.knn_classify(train, labels, test, test_labels=np.asarray(pred), k=int(k))
        np.testing.assert_array_equal(got, pred)
        assert acc == 1.0


@pytest.mark.gpu
def test_device_projection_large_sparse_fp32():
    # GP-SPCA-shaped: fp32 samples, sparse loadings (few active features)
    g = _gps()
    rng = np.random.default_rng(7)
    S = rng.standard_normal((3000, 5000)).astype(np.float32)
    L = sparse_loadings(8, 5000, 12, 40)
    A = g.DataMatrix(S)
    S64 = S.astype(np.float64)
    np.testing.assert_allclose(g.project(A, L), orc.embed(S64, L), rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(g.explained_variance(A, L), orc.variance_explained(S64, L), rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_device_knn_large_vs_oracle():
    g = _gps()
    rng = np.random.default_rng(11)
    train = rng.standard_normal((4000, 16))
    test = rng.standard_normal((2500, 16))
    labels = rng.integers(0, 10, 4000)
    for k in (1, 4):
        got, _ = g.knn_classify(train, labels, test, k=k)
        np.testing.assert_array_equal(got, orc.knn_predict(train, labels, test, k))


@pytest.mark.gpu
def test_device_recognition_errors():
    g = _gps()
    with pytest.raises(ValueError):
        g.project(np.ones((4, 3)), np.ones((2, 1)))
    with pytest.raises(ValueError):
        g.explained_variance(np.ones((4, 3)), 2.0 * np.eye(3)[:, :1])
    with pytest.raises(ValueError):
        g.knn_classify(np.ones((3, 2)), [0, 1, 2], np.ones((2, 2)), k=4)
    with pytest.raises(ValueError):
        g.knn_classify(np.zeros((0, 2)), [], np.ones((2, 2)))
    with pytest.raises(ValueError):
        g.pca_fit(np.ones((4, 3)), 5)


@pytest.mark.gpu
def test_device_center_columns_and_gram_quadratic():
    # core.py:234-256
    g = _gps()
    rng = np.random.default_rng(21)
    for dtype in (np.float64, np.float32):
        S = (rng.standard_normal((70, 45)) * 3 + 5).astype(dtype)
        C = g.center_columns(S)
        S64 = S.astype(np.float64)
        np.testing.assert_allclose(C.values, S64 - S64.mean(axis=0), rtol=0, atol=1e-12)
        assert C.dtype == np.float64 and C.shape == S.shape
        z = rng.standard_normal(45)
        v = S64 @ z
        assert g.gram_quadratic(S, z) == pytest.approx(float(v @ v), rel=1e-12)
    with pytest.raises(ValueError):
        g.gram_quadratic(np.ones((3, 4)), np.ones(3))


@pytest.mark.gpu
def test_fit_projection_centres_on_device():
    # bench.py:78-114 fit_projection: loadings of the centred training data
    from paper_1312_6182_b200.timing import fit_projection

    rng = np.random.default_rng(22)
    X = rng.standard_normal((80, 30)) + 2.0
    Z, mean, report = fit_projection(X, "sl1", 2, 0.05)
    np.testing.assert_allclose(mean, X.mean(axis=0), rtol=1e-12)
    assert Z.shape == (30, 2) and report.iterations >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1500, 200), (120, 700)], ids=["tall", "wide"])
def test_device_pca_fit_jacobi_both_orientations(shape):
    """pca_fit's device one-sided Jacobi SVD on both orientations (columns of
    S when n <= p, of S' otherwise) against pca.py:37-54 restated with
    LAPACK: top components with separated singular values."""
    g = _gps()
    rng = np.random.default_rng(5)
    N, F = shape
    S = rng.standard_normal((N, F)) @ np.diag(np.linspace(3.0, 1.0, F)) + 0.5
    model = g.pca_fit(S, 6)
    Sc = S - S.mean(axis=0)
    _, s, Vt = np.linalg.svd(Sc, full_matrices=False)
    np.testing.assert_allclose(model.singular_values, s[:6], rtol=1e-11)
    ref = g.recognition.deterministic_signs(Vt[:6].T)
    np.testing.assert_allclose(model.components, ref, atol=1e-8)
