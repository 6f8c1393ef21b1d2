"""Direction sharding with world_size 2 on CPU (gloo).

Also the far-field matvec (eq. (4) -> (5) -> (6), fmmt_far_matvec): each rank aggregates, translates and
disaggregates its own direction block; the all_reduce(SUM) of the per-rank y over ranks equals the
unsharded y (the reduction the library's ncclAllReduce of y performs).

The sharded translate_sum path partitions the plane-wave directions with the
library's `fmmt_shard_range` (pure host arithmetic) and allreduces the
weighted direction sum of eq. (6).  Here each gloo rank takes its
shard from the library, computes its partial sum with the ORACLE translation
(test infrastructure), and the all_reduce(SUM) over ranks must equal the
unsharded oracle sum: the decomposition the NCCL path relies on.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import translate
    from paper_2010_00520_b200 import fmmt
    from synth import config, signature_seed, signatures
    from tests._helpers import operator

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = config(1)
    T4, w, _ = operator(1)
    nd = T4.shape[-1]
    sig = signatures(signature_seed(1, 0), nd, c.Nx, c.Ny, c.Nz)
    b0, cnt = fmmt.shard_range(nd, rank, world)
    sig_m = translate.sig_to_math(sig)
    part = np.zeros((c.Nx, c.Ny, c.Nz), dtype=np.complex128)
    for p in range(b0, b0 + cnt):
        part += w[p] * translate.translate_fft(T4[..., p], sig_m[p])
    t = torch.from_numpy(np.stack([part.real, part.imag]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    counts = torch.tensor([cnt], dtype=torch.int64)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    if rank == 0:
        full = np.zeros_like(part)
        for p in range(nd):
            full += w[p] * translate.translate_fft(T4[..., p], sig_m[p])
        got = t[0].numpy() + 1j * t[1].numpy()
        q.put((float(np.linalg.norm(got - full) / np.linalg.norm(full)), int(counts.item()), nd))
    dist.destroy_process_group()


def _far_worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import aggregate
    from paper_2010_00520_b200 import fmmt
    from synth import basis, basis_seed, config, currents, patterns
    from tests._helpers import operator

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = config(1)
    T4, w, _ = operator(1)
    nd = T4.shape[-1]
    b = basis(basis_seed(1), c.Nx, c.Ny, c.Nz, c.edge)
    P = patterns(basis_seed(1) + 1, nd, b.N, 2)
    I = currents(basis_seed(1) + 2, b.N)
    b0, cnt = fmmt.shard_range(nd, rank, world)
    y = aggregate.far_matvec(P[b0:b0 + cnt], I, b.box_ptr, w[b0:b0 + cnt], lambda p: T4[..., b0 + p],
                             c.Nx, c.Ny, c.Nz)
    t = torch.from_numpy(np.stack([y.real, y.imag]))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    if rank == 0:
        full = aggregate.far_matvec(P, I, b.box_ptr, w, lambda p: T4[..., p], c.Nx, c.Ny, c.Nz)
        got = t[0].numpy() + 1j * t[1].numpy()
        q.put(float(np.linalg.norm(got - full) / np.linalg.norm(full)))
    dist.destroy_process_group()


def _run_two(target):
    import socket

    import torch.multiprocessing as mp
    from paper_2010_00520_b200 import build
    build.build()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_two_rank_far_matvec_shards_sum_to_unsharded():
    assert _run_two(_far_worker) < 1e-13


def test_two_rank_direction_shards_sum_to_unsharded():
    import socket

    import torch.multiprocessing as mp
    from paper_2010_00520_b200 import build
    build.build()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, total, nd = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert total == nd
    assert err < 1e-13
