"""The column-sharded driver with the device kernels (DeviceOps): one rank on
the GPU, and two gloo ranks sharing the GPU (host-mediated collectives, so no
rank's kernels wait on another's), against the single-process oracle."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import cnmf_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def _shard_job(rank, world, a32):
    import paper_1505_04650_b200 as C
    from paper_1505_04650_b200 import distributed as D
    from paper_1505_04650_b200.device import DeviceMatrix

    m, n = a32.shape
    c0, ni = D.column_shard(n, world, rank)
    A = DeviceMatrix(torch.from_numpy(np.ascontiguousarray(a32[:, c0: c0 + ni])).cuda())
    comm, ops = D.Comm(), D.DeviceOps()
    counts = [D.column_shard(n, world, k)[1] for k in range(world)]
    from dataclasses import replace

    cfg = C.adjust_config(C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), m, n)
    L = D.range_finder(ops, comm, A, m, n, c0, replace(cfg, seed=C.child_seed(5, "left-basis")), 0)
    R = comm.allgather_rows(D.range_finder(ops, comm, A, m, n, c0, replace(cfg, seed=C.child_seed(5, "right-basis")), 1),
                            counts)
    s = cfg.basis_cols
    u, vt_local, it, _, rel = D.nmf_admm(A, m, n, c0, 20, C.CompressionConfig(r=20, r_ov=10, w=4, seed=5), comm, ops,
                                         max_iter=500, tol=1e-4)
    # column-sharded SNMF on a near-separable instance (SPA and XRAY)
    sep = O.near_separable(3000, 1200, 12, 1.0, 0.005, seed=3)[0].astype(np.float32)
    ms, ns = sep.shape
    c0s, nis = D.column_shard(ns, world, rank)
    As = DeviceMatrix(torch.from_numpy(np.ascontiguousarray(sep[:, c0s: c0s + nis])).cuda())
    snmf = {}
    for sel in ("spa", "xray"):
        out = D.snmf(ops, comm, As, ms, ns, c0s, 12, selector=sel, cfg=C.CompressionConfig(r=12, r_ov=10, w=2, seed=9),
                     host_out=True)
        snmf[sel] = (out.K, out.Y, out.rel_error_full)
    torch.cuda.synchronize()
    return (L[:, :s].double().cpu().numpy(), R[:, :s].double().cpu().numpy(), it, rel, snmf)


def _worker(rank, world, port, a32, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _shard_job(rank, world, a32)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def problem():
    a32 = O.dense_lowrank(2000, 1001, 20, 0.01, seed=0).astype(np.float32)
    a = a32.astype(np.float64)
    cfg = O.adjust(O.Config(20, 10, 4, 5), *a.shape)
    from dataclasses import replace

    L = O.range_basis(a, replace(cfg, seed=O.child_seed(5, "left-basis")))
    R = O.row_basis(a, replace(cfg, seed=O.child_seed(5, "right-basis")))
    ref = O.admm(a, 20, cfg=O.Config(20, 10, 4, 5), max_iter=500, tol=1e-4)
    # the reference's own spread when the input is perturbed at fp32 level
    # (2^-23 relative): the yardstick for a device run whose passes are fp32
    rng = np.random.default_rng(0)
    spread = 0.0
    for _ in range(3):
        o = O.admm(a * (1.0 + 2.0 ** -23 * rng.standard_normal(a.shape)), 20, cfg=O.Config(20, 10, 4, 5),
                   max_iter=500, tol=1e-4)
        spread = max(spread, abs(O.rel_error(a, o.X, o.Y) - ref.rel_error))
    # the reference's own subspace band under one fp32 rounding of A (2^-24)
    band = 0.0
    for k in range(2):
        ap = a * (1.0 + 2.0 ** -24 * np.random.default_rng(10 + k).standard_normal(a.shape))
        band = max(band, O.projector_distance(L, O.range_basis(ap, replace(cfg, seed=O.child_seed(5, "left-basis")))),
                   O.projector_distance(R, O.row_basis(ap, replace(cfg, seed=O.child_seed(5, "right-basis")))))
    return a32, L, R, ref, (spread, band)


def _check(res, problem):
    a32, L, R, ref, (spread, band) = problem
    Ld, Rd, it, rel, snmf = res
    sig = slice(0, 20)
    assert O.projector_distance(L[:, sig], Ld[:, sig]) < 1e-5
    assert O.projector_distance(R[:, sig], Rd[:, sig]) < 1e-5
    # full basis: north-star 1e-4, or twice the reference's own movement under
    # one fp32 rounding of A (tests/test_gpu_fullsize.py)
    assert O.projector_distance(L, Ld) <= max(1e-4, 2.0 * band)
    assert O.projector_distance(R, Rd) <= max(1e-4, 2.0 * band)
    assert it == ref.iterations
    sep = O.near_separable(3000, 1200, 12, 1.0, 0.005, seed=3)[0].astype(np.float32).astype(np.float64)
    for sel, (K, Y, rf) in snmf.items():
        o = O.snmf(sep, 12, selector=sel, cfg=O.Config(12, 10, 2, 9))
        np.testing.assert_array_equal(K, o.K)
        assert abs(rf - o.rel_error_full) <= 1e-3 * o.rel_error_full
        assert np.abs(Y - o.Y).max() <= 1e-3 * max(1.0, np.abs(o.Y).max())
    # the ADMM amplifies input perturbations over 500 iterations:
    # within 2e-3 relative, or within 3x the reference's own spread under
    # fp32-level input perturbations
    assert abs(rel - ref.rel_error) <= max(2e-3 * ref.rel_error, 3.0 * spread)


def test_sharded_driver_one_rank(problem):
    _check(_shard_job(0, 1, problem[0]), problem)


def test_sharded_driver_two_gloo_ranks_on_one_gpu(problem):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, problem[0], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    _check(res, problem)
