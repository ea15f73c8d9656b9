"""Plane summaries and transfer-matrix metrics (holopipe/analysis.py).

The per-frame reductions run on the GPU (``hpg_run`` with HPG_FLAG_SUMMARY,
``hpg_plane_summary``, ``hpg_metric_partials``).  What is left for the host is
the O(rows + cols^2) finish of the nine metrics from the fp64 partial sums:
logarithms, extrema, and the eigenvalues of the (small) Gram matrix for MDL,
mirroring holopipe/analysis.py:143-188.  Partials from several GPUs are summed
(NCCL all-reduce / all-gather) before this finish.
"""

from __future__ import annotations

import math

import numpy as np

from . import constants as C

SNR_CAP_DB = 200.0
_NEG = float(np.finfo(np.float32).min)


class AnalysisSummary:
    """parameters (ANALYSIS_COUNT, polCount, totalCount) float32, summed intensity, axes."""

    def __init__(self, parameters, total_intensity, x_axis, y_axis, plane):
        self.parameters = parameters
        self.total_intensity = total_intensity
        self.x_axis = x_axis
        self.y_axis = y_axis
        self.plane = plane


def analysis_value(summary, param, pol, idx):
    v = summary.parameters[param, pol, idx]
    if param == C.ANALYSIS_MAXABSIDX:
        return int(np.float32(v).view(np.int32))
    return float(v)


class MetricsReport:
    """values (METRIC_COUNT, wavelengthCount+1) float32; last slot = average."""

    def __init__(self, wavelength_count=1):
        self.wavelength_count = int(wavelength_count)
        self.values = np.full((C.METRIC_COUNT, self.wavelength_count + 1), C.METRIC_UNSET,
                              dtype=np.float32)
        self._mdl_pending = None   # [(slot, gram, nd)]: MDL eigenvalues computed on first read

    def defer_mdl(self, pending):
        """MDL needs the eigenvalues of each wavelength's Gram matrix (~0.1-0.2 ms of LAPACK for 45 modes);
        AutoAlign reads only its goal metric per evaluation, so the decomposition runs on the first read
        of METRIC_MDL instead of inside every calc_metrics."""
        self._mdl_pending = list(pending) or None

    def _resolve(self, idx):
        if idx != C.METRIC_MDL or self._mdl_pending is None:
            return
        L = self.wavelength_count
        row = np.full(L, C.METRIC_UNSET, np.float64)
        for w, gram, nd in self._mdl_pending:
            row[w] = mdl_db(gram, nd)
            self.values[C.METRIC_MDL, w] = np.float32(row[w])
        self._mdl_pending = None
        ok = row[row > C.METRIC_UNSET / 2]
        self.values[C.METRIC_MDL, L] = np.float32(ok.mean()) if ok.size else C.METRIC_UNSET

    def get(self, idx):
        if not (0 <= idx < C.METRIC_COUNT):
            return 0.0
        self._resolve(idx)
        return float(self.values[idx, self.wavelength_count])

    def get_all(self, idx):
        if not (0 <= idx < C.METRIC_COUNT):
            return None
        self._resolve(idx)
        return self.values[idx].copy()


def _db(x):
    return _NEG if x <= 0 else 10.0 * math.log10(x)


def _snr(sig, noise):
    if sig <= 0:
        return _NEG
    if noise <= 0:
        return SNR_CAP_DB
    return min(10.0 * math.log10(sig / noise), SNR_CAP_DB)


def _snr_of_ratio(r):
    """Per-row SNR in dB from signal / noise (0: no signal -> unset; inf: no noise -> cap)."""
    if r <= 0:
        return _NEG
    if math.isinf(r):
        return SNR_CAP_DB
    return min(float(10.0 * np.log10(r)), SNR_CAP_DB)


def mdl_db(gram, nd):
    """MDL = 10 log10(lambda_max / lambda_min) over the top min(rows, cols) eigenvalues of the Gram matrix
    (the squared singular values; holopipe/analysis.py:158-162 takes an SVD of the matrix itself)."""
    ev = np.linalg.eigvalsh(np.asarray(gram, np.complex128))
    top = ev[-nd:]
    lo, hi = float(top.min()), float(top.max())
    return 10.0 * math.log10(hi / lo) if lo > 0 else C.METRIC_UNSET


def finish_metrics(row_power, diag_power, group_power, gram, rows, cols, have_labels=True, defer_mdl=False):
    """Nine metrics from fp64 partials of one transfer matrix (analysis.py:143-188).

    row_power/diag_power/group_power are per virtual row (diag entries < 0 mark
    rows without a diagonal element); gram is the Hermitian Gram matrix whose
    top min(rows, cols) eigenvalues are the squared singular values.
    """
    v = np.full(C.METRIC_COUNT, C.METRIC_UNSET, dtype=np.float64)
    if rows == 0 or cols == 0:
        return v
    row_power = np.asarray(row_power, np.float64)
    nd = min(rows, cols)
    has = np.asarray(diag_power) >= 0
    d = np.asarray(diag_power, np.float64)[has][:nd]
    grp = np.asarray(group_power, np.float64)[has][:nd]
    rowd = row_power[has][:nd]
    total = float(row_power.sum())
    v[C.METRIC_IL] = _db(float(row_power.mean()))
    if total > 0 and gram is not None and not defer_mdl:
        v[C.METRIC_MDL] = mdl_db(gram, nd)
    dt = float(d.sum())
    v[C.METRIC_DIAG] = _db(dt / nd)
    v[C.METRIC_SNRAVG] = _snr(dt, total - dt)
    # best / worst per-row values: 10 log10 is monotonic, so take the extrema first and convert two scalars
    # (the per-row rules of analysis.py:165-176: d <= 0 -> unset, no noise -> cap)
    dmax, dmin = float(d.max()), float(d.min())
    v[C.METRIC_DIAGBEST] = float(10.0 * np.log10(dmax)) if dmax > 0 else _NEG
    v[C.METRIC_DIAGWORST] = float(10.0 * np.log10(dmin)) if dmin > 0 else _NEG
    noise = rowd - d
    ratio = np.where(d > 0, np.where(noise > 0, d / np.where(noise > 0, noise, 1.0), np.inf), 0.0)
    v[C.METRIC_SNRBEST] = _snr_of_ratio(float(ratio.max()))
    v[C.METRIC_SNRWORST] = _snr_of_ratio(float(ratio.min()))
    if have_labels:
        sig = float(grp.sum())
        v[C.METRIC_SNRMG] = _snr(sig, total - sig)
    else:
        v[C.METRIC_SNRMG] = v[C.METRIC_SNRAVG]
    return v


def metrics_of_matrix(A, labels=None):
    """Host metrics of an explicit complex matrix (used for A A^H, analysis.py:124-125)."""
    A = np.asarray(A, np.complex128)
    pw = np.abs(A) ** 2
    R, Cc = A.shape
    nd = min(R, Cc)
    rp = pw.sum(axis=1)
    d = np.full(R, -1.0)
    d[:nd] = pw[np.arange(nd), np.arange(nd)]
    grp = d.copy()
    if labels is not None:
        lab = np.asarray(labels)
        grp[:nd] = np.where(lab[:nd, None] == lab[None, :], pw[:nd], 0.0).sum(axis=1)
    gram = A @ A.conj().T if R <= Cc else A.conj().T @ A
    return finish_metrics(rp, d, grp, gram, R, Cc, labels is not None)


def average_slot(per_wl):
    """Across-wavelength mean of valid values (analysis.py:243-247)."""
    per_wl = np.asarray(per_wl, np.float64)
    L = per_wl.shape[1]
    rep = MetricsReport(L)
    rep.values[:, :L] = per_wl.astype(np.float32)
    if L == 1:   # the average of one valid value is the value
        ok = per_wl[:, 0] > C.METRIC_UNSET / 2
        rep.values[ok, 1] = per_wl[ok, 0].astype(np.float32)
        return rep
    for m in range(C.METRIC_COUNT):
        ok = per_wl[m][per_wl[m] > C.METRIC_UNSET / 2]
        if ok.size:
            rep.values[m, L] = np.float32(ok.mean())
    return rep
