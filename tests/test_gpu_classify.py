"""Batched Classifier::predict on the B200 path through the C ABI
(rbd_classify_batch) against the oracle's restatement of classify.cpp:22-34 and
the reference's own classify tests (test_classify.cpp:31-131, test_smoke.py:74-79).
Parity: the chosen training column equals the oracle's, except where the oracle's
two smallest distances lie within 1e-12 (relative) of each other (summation order)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1503_05947_b200 as rbd

pytestmark = pytest.mark.gpu


def check_parity(clf, queries):
    got = clf.predict_indices(queries)
    Yh = clf.model.Y.cpu().numpy() if hasattr(clf.model.Y, "cpu") else clf.model.Y
    Th = clf.model.T.cpu().numpy() if hasattr(clf.model.T, "cpu") else clf.model.T
    qh = queries.cpu().numpy() if hasattr(queries, "cpu") else np.asarray(queries)
    ref, rdist = oracle.predict_batch(Yh, Th, qh, nthreads=8)
    diff = np.nonzero(got != ref)[0]
    for q in diff:   # admissible only as a near tie
        c = Yh.T @ qh[:, q]
        d_got = ((Th[:, got[q]] - c) ** 2).sum()
        assert abs(d_got - rdist[q]) <= 1e-12 * max(rdist[q], 1e-300), (q, d_got, rdist[q])
    return got, len(diff)


def labels_of(ids):
    return [str(int(i)) for i in ids]


def test_well_separated_clusters_classify_perfectly(cuda):        # test_classify.cpp:31-51
    samples, lab = oracle.gen_labeled_blobs(5, 18, 30, 0.01, 800)
    tr = [c * 18 + k for c in range(5) for k in range(10)]
    te = [c * 18 + k for c in range(5) for k in range(10, 18)]
    clf = rbd.fit(samples[:, tr], labels_of(lab[tr]), d_max=10)
    assert clf.evaluate(samples[:, te], labels_of(lab[te])) == 0.0
    check_parity(clf, samples[:, te])


def test_predict_equals_brute_force(cuda):                         # test_classify.cpp:53-75
    train = oracle.random_matrix(20, 15, 810)
    labels = ["c" + str(j % 4) for j in range(15)]
    clf = rbd.fit(train, labels, d_max=6)
    queries = oracle.random_matrix(20, 12, 811)
    got, _ = check_parity(clf, queries)
    for q in range(12):
        c = clf.model.Y.T @ queries[:, q]
        dist = ((clf.train_coords - c[:, None]) ** 2).sum(axis=0)
        assert clf.predict(queries[:, q]) == labels[int(np.argmin(dist))]


def test_ties_resolve_to_the_earliest_column(cuda):               # test_classify.cpp:77-89
    train = np.zeros((4, 3))
    train[0, 0] = train[0, 1] = 1.0
    train[1, 2] = 1.0
    clf = rbd.fit(train, ["first", "second", "other"], d_max=2)
    assert clf.predict(np.array([1.0, 0.1, 0.0, 0.0])) == "first"


def test_orthogonal_components_are_ignored(cuda):                 # test_classify.cpp:91-103
    train = oracle.random_matrix(25, 12, 820)
    clf = rbd.fit(train, [str(j % 3) for j in range(12)], d_max=5)
    v = oracle.random_matrix(25, 1, 821)[:, 0]
    w = oracle.random_matrix(25, 1, 822)[:, 0]
    w -= clf.model.Y @ (clf.model.Y.T @ w)
    assert clf.predict(v) == clf.predict(v + 10.0 * w)


def test_validation(cuda):                                        # test_classify.cpp:105-131
    with pytest.raises(rbd.DimensionMismatch):
        rbd.fit(oracle.random_matrix(8, 5, 830), ["a", "b"], d_max=2)
    train = oracle.random_matrix(6, 4, 840)
    clf = rbd.fit(train, ["a", "a", "b", "b"], d_max=3)
    with pytest.raises(rbd.DimensionMismatch):
        clf.evaluate(oracle.random_matrix(5, 2, 841), ["a", "b"])
    with pytest.raises(rbd.DimensionMismatch):
        clf.evaluate(oracle.random_matrix(6, 2, 842), ["a"])
    assert clf.evaluate(train, ["a", "a", "b", "b"]) == 0.0
    assert clf.evaluate(train, ["b", "b", "a", "a"]) == 1.0


def test_smoke_blobs(cuda):                                       # test_smoke.py:74-79
    samples, lab = oracle.gen_labeled_blobs(3, 10, 16, 0.05, 5)
    names = labels_of(lab)
    clf = rbd.fit(samples, names, d_max=8)
    assert clf.predict(samples[:, 0]) == names[0]


@pytest.mark.parametrize("m,n_tr,d,nq", [(300, 1000, 40, 777), (4096, 2432, 129, 3000),
                                         (65, 64, 64, 64), (33, 5, 3, 1), (1000, 130, 17, 65)])
def test_parity_random_shapes(cuda, m, n_tr, d, nq):
    rng = np.random.default_rng(m + n_tr)
    train = rng.standard_normal((m, n_tr))
    clf = rbd.fit(train, [str(j) for j in range(n_tr)], d_max=d)
    queries = train[:, rng.integers(0, n_tr, nq)] + 0.3 * rng.standard_normal((m, nq))
    check_parity(clf, queries)


def test_device_resident_model_and_queries(cuda):
    g = torch.Generator(device="cuda").manual_seed(3)
    m, n_tr, nq = 8192, 3000, 5000
    X = torch.randn(n_tr, m, generator=g, device="cuda", dtype=torch.float64).t()
    clf = rbd.fit(X, [str(j) for j in range(n_tr)], d_max=200)
    src = torch.arange(nq, device="cuda") % n_tr
    Q = X[:, src] + 0.05 * torch.randn(m, nq, generator=g, device="cuda", dtype=torch.float64)
    Q = Q.t().contiguous().t()
    got, _ = check_parity(clf, Q)
    assert (got == (np.arange(nq) % n_tr)).mean() > 0.99   # nearest to its own source column
