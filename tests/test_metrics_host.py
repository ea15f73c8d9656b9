"""Host-side metric finishing (CPU): the deferred MDL of MetricsReport equals the eager value, and the
finishing matches the oracle's restatement of holopipe/analysis.py:104-248 on the same matrices."""

import numpy as np
import pytest

from oracle import holo_oracle as O
from paper_2204_02348_b200 import constants as C
from paper_2204_02348_b200.analysis import average_slot, finish_metrics, mdl_db, metrics_of_matrix


def _partials(A, labels):
    pw = np.abs(A) ** 2
    R, Cc = A.shape
    nd = min(R, Cc)
    d = np.full(R, -1.0)
    d[:nd] = pw[np.arange(nd), np.arange(nd)]
    grp = d.copy()
    grp[:nd] = np.where(labels[:nd, None] == labels[None, :], pw[:nd], 0.0).sum(axis=1)
    gram = A @ A.conj().T if R <= Cc else A.conj().T @ A
    return pw.sum(axis=1), d, grp, gram


@pytest.mark.parametrize("shape", [(45, 45), (128, 45), (20, 45)])
def test_deferred_mdl_equals_eager(rng, shape):
    L = 2
    per = np.full((C.METRIC_COUNT, L), C.METRIC_UNSET)
    pending, eager = [], []
    for w in range(L):
        A = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        labels = np.array([O.group_of_mode(i) for i in range(shape[1])])
        rp, d, grp, gram = _partials(A, labels)
        v_eager = finish_metrics(rp, d, grp, gram, shape[0], shape[1], True)
        v_def = finish_metrics(rp, d, grp, gram, shape[0], shape[1], True, defer_mdl=True)
        assert v_def[C.METRIC_MDL] == C.METRIC_UNSET
        mask = np.arange(C.METRIC_COUNT) != C.METRIC_MDL
        assert np.array_equal(v_eager[mask], v_def[mask])
        per[:, w] = v_def
        pending.append((w, gram, min(shape)))
        eager.append(v_eager)
    rep = average_slot(per)
    rep.defer_mdl(pending)
    ref = average_slot(np.stack(eager, axis=1))
    for m in range(C.METRIC_COUNT):
        assert np.array_equal(rep.get_all(m), ref.get_all(m)), m
    assert rep.get(C.METRIC_MDL) == ref.get(C.METRIC_MDL)


def test_metrics_match_oracle_restatement(rng):
    A = rng.standard_normal((60, 45)) + 1j * rng.standard_normal((60, 45))
    labels = np.array([O.group_of_mode(i) for i in range(45)])
    v = metrics_of_matrix(A, labels)
    ref = np.asarray(O.metrics_one(A, labels), np.float64)
    assert np.allclose(v, ref, rtol=0, atol=1e-6)


def test_mdl_of_rank_deficient_matrix_is_unset():
    A = np.zeros((10, 10), np.complex128)
    A[0, 0] = 1.0
    assert mdl_db(A.conj().T @ A, 10) == C.METRIC_UNSET
