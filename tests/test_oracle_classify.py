"""Pins the oracle's Classifier restatement (classify.cpp:11-48) to the reference's
own tests (proj/tests/test_classify.cpp:31-131, python/test_smoke.py:74-79)."""
import numpy as np

import oracle


def fit(train, d):
    return oracle.decompose(train, d)


def predict(model, v):
    best, _ = oracle.predict_batch(model.Y, model.T, v)
    return best


def test_well_separated_clusters_classify_perfectly():            # test_classify.cpp:31-51
    samples, lab = oracle.gen_labeled_blobs(5, 18, 30, 0.01, 800)
    tr = [c * 18 + k for c in range(5) for k in range(10)]
    te = [c * 18 + k for c in range(5) for k in range(10, 18)]
    model = fit(samples[:, tr], 10)
    best = predict(model, samples[:, te])
    assert np.array_equal(lab[tr][best], lab[te])


def test_predict_equals_brute_force_nearest_neighbour():           # test_classify.cpp:53-75
    train = oracle.random_matrix(20, 15, 810)
    model = fit(train, 6)
    queries = oracle.random_matrix(20, 12, 811)
    best = predict(model, queries)
    for q in range(12):
        c = model.Y.T @ queries[:, q]
        dist = ((model.T - c[:, None]) ** 2).sum(axis=0)
        assert best[q] == int(np.argmin(dist))


def test_ties_resolve_to_the_earliest_column():                   # test_classify.cpp:77-89
    train = np.zeros((4, 3))
    train[0, 0] = train[0, 1] = 1.0
    train[1, 2] = 1.0
    model = fit(train, 2)
    assert predict(model, np.array([1.0, 0.1, 0.0, 0.0]))[0] == 0


def test_components_orthogonal_to_the_basis_are_ignored():        # test_classify.cpp:91-103
    train = oracle.random_matrix(25, 12, 820)
    model = fit(train, 5)
    v = oracle.random_matrix(25, 1, 821)[:, 0]
    w = oracle.random_matrix(25, 1, 822)[:, 0]
    w -= model.Y @ (model.Y.T @ w)
    assert predict(model, v)[0] == predict(model, v + 10.0 * w)[0]


def test_smoke_blobs():                                           # test_smoke.py:74-79
    samples, lab = oracle.gen_labeled_blobs(3, 10, 16, 0.05, 5)
    model = fit(samples, 8)
    assert lab[predict(model, samples[:, 0])[0]] == lab[0]
