"""Multi-GPU data parallelism over frames.

Frames (batch rows) are independent for fields and coefficients, so each
rank processes a contiguous shard of the batch with its own engine and plan
replica -- no collective on the data path.  The only exchange is the metric
reduction AutoAlign iterates on: each rank computes fp64 partials of its
rows on the GPU (hpg_metric_partials), then

  * the Gram matrix A^H A (cols x cols) is all-reduced (sum),
  * the per-row power / diagonal / mode-group sums are all-gathered,

and every rank finishes the nine metrics identically on the host
(analysis.finish_metrics), so AutoAlign decisions stay replicated and
deterministic.  Works with NCCL (GPU tensors) and gloo (CPU tensors, used by
the CPU tests).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import constants as C
from .analysis import average_slot, finish_metrics
from .engine import mode_group_of_index


def shard(batch, world, rank):
    """Contiguous [start, stop) rows of ``batch`` owned by ``rank``."""
    per = -(-batch // world)
    start = min(batch, rank * per)
    return start, min(batch, start + per)


def _all_gather_var(t, group=None):
    """all_gather of 1-D tensors of different lengths, concatenated in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(mx, dtype=t.dtype, device=t.device)
    buf[:t.numel()] = t
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[:int(s.item())] for o, s in zip(out, sizes)])


def exclusive_prefix(count, group=None, device="cpu"):
    """Sum of ``count`` over lower ranks (global row offset of this shard)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([int(count)], dtype=torch.int64, device=device)
    all_c = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(all_c, t, group=group)
    r = dist.get_rank(group)
    return int(sum(int(c.item()) for c in all_c[:r])), int(sum(int(c.item()) for c in all_c))


def reduce_and_finish(row_power, diag_power, group_power, gram, rows_global, cols, group=None,
                      have_labels=True, defer_mdl=False):
    """Combine per-rank partials (torch tensors on the process-group device) into the metrics.

    ``defer_mdl``: leave METRIC_MDL unset and return the reduced Gram matrix as well (the eigenvalue
    problem runs only when MDL is read, as the engine does for AutoAlign, analysis.MetricsReport.defer_mdl)."""
    import torch.distributed as dist
    dist.all_reduce(gram, group=group)
    rp = _all_gather_var(row_power, group).cpu().numpy()
    dp = _all_gather_var(diag_power, group).cpu().numpy()
    gp = _all_gather_var(group_power, group).cpu().numpy()
    g = gram.cpu().numpy()
    v = finish_metrics(rp, dp, gp, g, rows_global, cols, have_labels, defer_mdl=defer_mdl)
    return (v, g) if defer_mdl else v


def host_partials(coefs, labels, diag_offset, ndiag):
    """Reference partial sums of one shard in numpy (what hpg_metric_partials computes)."""
    A = np.asarray(coefs, np.complex128)
    pw = np.abs(A) ** 2
    R, Cc = A.shape
    rp = pw.sum(axis=1)
    dp = np.full(R, -1.0)
    gp = np.full(R, -1.0)
    for r in range(R):
        d = r + diag_offset
        if d < ndiag:
            dp[r] = pw[r, d]
            gp[r] = pw[r, np.asarray(labels) == labels[d]].sum() if labels is not None else dp[r]
    gram = A.conj().T @ A
    return rp, dp, gp, gram


def shard_partials(coefs, local_rows, labels, diag_offset, ndiag, dev):
    """fp64 partial sums of one shard's rows of one wavelength, on the GPU (hpg_metric_partials).

    ``local_rows``: indices into ``coefs`` (this rank's rows of the wavelength, in global order);
    ``diag_offset``: the global index, among the wavelength's rows, of the first of them -- the
    transfer-matrix diagonal runs along the GLOBAL row (holopipe/analysis.py:155-176);
    ``ndiag``: min(global rows of the wavelength, cols).  Returns (row, diag, group power, Gram)."""
    import torch
    from . import native
    R = len(local_rows)
    cols = coefs.shape[1]
    rp = torch.zeros(R, dtype=torch.float64, device=dev)
    dp = torch.full((R,), -1.0, dtype=torch.float64, device=dev)
    gp = torch.full((R,), -1.0, dtype=torch.float64, device=dev)
    gram = torch.zeros((cols, cols), dtype=torch.complex128, device=dev)
    big = R * cols * cols > (1 << 28)   # large shards: the Gram A^H A is a plain library GEMM (cuBLAS zgemm)
    if R:
        ids = torch.as_tensor(np.asarray(local_rows, np.int32), device=dev)
        a = native.MetricArgs()
        a.coefs = coefs.data_ptr()
        a.rows, a.cols, a.ld = R, cols, cols
        a.row_ids = ids.data_ptr()
        a.labels = labels.data_ptr()
        a.ndiag, a.diag_offset, a.gram_rows = ndiag, diag_offset, 0
        a.row_power, a.diag_power, a.group_power = rp.data_ptr(), dp.data_ptr(), gp.data_ptr()
        a.gram = None if big else gram.data_ptr()
        with torch.cuda.device(dev):
            native.check(native.lib().hpg_metric_partials(ctypes.byref(a), native.stream_handle(dev)),
                         "hpg_metric_partials")
            if big:
                gram_of_rows(coefs, ids.long(), gram)
    return rp, dp, gp, gram


def gram_of_rows(coefs, ids, out, chunk=8192):
    """out[i][j] = sum_k A[k][i] conj(A[k][j]) for A = coefs[ids] in complex128 -- the MDL Gram exactly as
    hpg_metric_partials lays it out (analysis.py:158-162; conj(A^H A), same eigenvalues) -- accumulated over
    row chunks with cuBLAS zgemm."""
    import torch
    for s0 in range(0, ids.numel(), chunk):
        A = coefs.index_select(0, ids[s0:s0 + chunk]).to(torch.complex128)
        out.addmm_(A.T, A.conj())
    return out


def mode_labels(P, M, dev):
    """(pol, mode group) label of every coefficient column: SNRMG's signal set (analysis.py:180-188)."""
    import torch
    return torch.as_tensor(np.array([q * 1000 + mode_group_of_index(i) for q in range(P) for i in range(M)],
                                    np.int32), device=dev)


def wavelength_of_rows(rows, B, cfg):
    """Wavelength index of global rows (holopipe/engine.py:102-106)."""
    L = len(cfg.wavelength_list())
    if cfg.wavelengthOrdering[C.WAVELENGTHORDER_INPUT] == C.WAVELENGTHORDER_FAST or L <= 1:
        return rows % L
    return np.minimum(rows * L // B, L - 1)


def calc_metrics(eng, group=None, defer_mdl=False):
    """Transfer-matrix metrics of a batch sharded over the process group.

    ``eng`` holds this rank's rows (a contiguous shard; its global row offset is the
    sum of the lower ranks' row counts); wavelength membership follows the global
    row index (holopipe/engine.py:102-106).  Returns the MetricsReport, identical on
    every rank.  Pol-independent / A A^H variants are single-process only.  ``defer_mdl``: MDL is
    resolved from the reduced Gram matrices on its first read (MetricsReport.defer_mdl).
    """
    cfg = eng.config
    dev = eng.device
    coefs = eng.coefs_device()
    B_local = coefs.shape[0]
    P, M = eng._st0["P"], eng._mode_count
    cols = P * M
    L = len(cfg.wavelength_list())
    start, B = exclusive_prefix(B_local, group, device=dev)
    wl = wavelength_of_rows(np.arange(start, start + B_local), B, cfg)
    labels = mode_labels(P, M, dev)
    per = np.full((C.METRIC_COUNT, L), C.METRIC_UNSET)
    pending = []
    for w in range(L):
        local = np.nonzero(wl == w)[0]
        off, n_w = exclusive_prefix(local.size, group, device=dev)
        if n_w == 0:
            continue
        rp, dp, gp, gram = shard_partials(coefs, local, labels, off, min(n_w, cols), dev)
        out = reduce_and_finish(rp, dp, gp, gram, n_w, cols, group, defer_mdl=defer_mdl)
        if defer_mdl:
            per[:, w], g = out
            pending.append((w, g, min(n_w, cols)))
        else:
            per[:, w] = out
    rep = average_slot(per)
    if defer_mdl:
        rep.defer_mdl(pending)
    return rep
