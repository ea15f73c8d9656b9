"""The multi-GPU metric path on hardware: hpg_metric_partials per shard with diag_offset != 0, then the
NCCL reduction (distributed.reduce_and_finish over a world-1 NCCL group), against the unsharded engine
and the reference's own metrics (holopipe/analysis.py:104-248; the diagonal is indexed by the GLOBAL row,
analysis.py:155-176).  A 1-GPU box cannot run two NCCL ranks, so the two shards' partials are combined
exactly as the all-reduce (Gram sum) and all-gather (row sums, rank order) would combine them."""
import socket

import numpy as np
import pytest

from tests.golden_util import load

pytestmark = pytest.mark.gpu
METRIC_TOL_DB = 1e-3


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    yield
    dist.destroy_process_group()


def _engine(name):
    from paper_2204_02348_b200.engine import Engine
    case, g, frames = load(name)
    eng = Engine()
    for k, v in case["config"].items():
        setattr(eng.config, k, v)
    eng.source.set_float32(frames)
    eng.run_pipeline(0)
    return eng, g


@pytest.mark.parametrize("name,split", [("pr1", 1), ("pr1", 3), ("dualpol", 1), ("multiwl", 3), ("largebasis", 1)])
def test_two_shard_metrics_match_unsharded_and_reference(nccl_world1, name, split):
    import torch
    from paper_2204_02348_b200 import constants as C
    from paper_2204_02348_b200 import distributed as D
    from paper_2204_02348_b200.analysis import average_slot
    eng, g = _engine(name)
    eng.calc_metrics()
    single = np.stack([eng.metrics_array(i) for i in range(C.METRIC_COUNT)])
    coefs = eng.coefs_device()
    B, cols = coefs.shape
    P, M = eng._st0["P"], eng._mode_count
    dev = eng.device
    labels = D.mode_labels(P, M, dev)
    wl = D.wavelength_of_rows(np.arange(B), B, eng.config)
    L = len(eng.config.wavelength_list())
    shards = [(0, split), (split, B)]
    per = np.full((C.METRIC_COUNT, L), C.METRIC_UNSET)
    offsets_seen = []
    for w in range(L):
        rows_w = [np.nonzero(wl[a:b] == w)[0] + a for a, b in shards]
        n_w = sum(r.size for r in rows_w)
        parts, off = [], 0
        for (a, b), rows in zip(shards, rows_w):
            # each "rank" holds coefs[a:b] only: local indices, global diagonal offset
            local = coefs[a:b].contiguous()
            parts.append(D.shard_partials(local, rows - a, labels, off, min(n_w, cols), dev))
            offsets_seen.append(off)
            off += rows.size
        rp = torch.cat([p[0] for p in parts])
        dp = torch.cat([p[1] for p in parts])
        gp = torch.cat([p[2] for p in parts])
        gram = parts[0][3] + parts[1][3]
        per[:, w] = D.reduce_and_finish(rp, dp, gp, gram, n_w, cols)   # NCCL all-reduce / all-gather
    sharded = np.stack([average_slot(per).get_all(i) for i in range(C.METRIC_COUNT)])
    assert max(offsets_seen) > 0, "no shard exercised a non-zero diag_offset"
    assert np.allclose(sharded, single, atol=METRIC_TOL_DB, rtol=0), np.abs(sharded - single).max()
    assert np.allclose(sharded, g["metrics"], atol=METRIC_TOL_DB, rtol=0), np.abs(sharded - g["metrics"]).max()


def test_calc_metrics_over_nccl_world1(nccl_world1):
    """distributed.calc_metrics end to end through NCCL (one rank holds the whole batch)."""
    from paper_2204_02348_b200 import constants as C
    from paper_2204_02348_b200 import distributed as D
    eng, g = _engine("multiwl")
    rep = D.calc_metrics(eng)
    got = np.stack([rep.get_all(i) for i in range(C.METRIC_COUNT)])
    assert np.allclose(got, g["metrics"], atol=METRIC_TOL_DB, rtol=0), np.abs(got - g["metrics"]).max()


def test_large_shard_gram_by_library_gemm_matches_native_kernel():
    """Shards with rows * cols^2 > 2^28 take the MDL Gram from cuBLAS zgemm (distributed.gram_of_rows);
    it equals hpg_metric_partials' own fp64 Gram kernel."""
    import ctypes
    import torch
    from paper_2204_02348_b200 import distributed as D
    from paper_2204_02348_b200 import native
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device="cpu").manual_seed(7)
    R, cols = 2100, 360
    coefs = torch.complex(torch.randn(R, cols, generator=g), torch.randn(R, cols, generator=g)).to(dev)
    labels = D.mode_labels(1, cols, dev)
    rows = np.arange(R)
    rp, dp, gp, gram = D.shard_partials(coefs, rows, labels, 0, cols, dev)   # big: library GEMM
    assert R * cols * cols > (1 << 28)
    ref = torch.zeros((cols, cols), dtype=torch.complex128, device=dev)
    ids = torch.as_tensor(rows.astype(np.int32), device=dev)
    a = native.MetricArgs()
    a.coefs, a.rows, a.cols, a.ld = coefs.data_ptr(), R, cols, cols
    a.row_ids, a.labels = ids.data_ptr(), labels.data_ptr()
    a.ndiag, a.diag_offset, a.gram_rows = cols, 0, 0
    tmp = torch.zeros(3 * R, dtype=torch.float64, device=dev)
    a.row_power, a.diag_power, a.group_power = tmp.data_ptr(), tmp.data_ptr() + 8 * R, tmp.data_ptr() + 16 * R
    a.gram = ref.data_ptr()
    native.check(native.lib().hpg_metric_partials(ctypes.byref(a), native.stream_handle(dev)), "partials")
    torch.cuda.synchronize()
    assert torch.allclose(gram, ref, rtol=1e-10, atol=1e-9 * ref.abs().max().item())
    assert torch.allclose(rp, tmp[:R])
