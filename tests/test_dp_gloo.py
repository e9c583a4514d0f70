"""N>1 data-parallel logic on CPU with the gloo backend (world size 2): the
sharded batch evaluation must equal the single-rank evaluation bit-exactly,
and timing is reduced as the max over ranks.  The per-shard compute here is
the C oracle (test infrastructure); on GPUs bench.py runs the same helpers
over NCCL with the sm_100a library."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_13055_b200 import dp

N, L, A, DB, LEVEL = 256, 6, 2, 48, 6


def _oracle_hmult_batch(x: torch.Tensor, y: torch.Tensor, evk: np.ndarray) -> torch.Tensor:
    from pyoracle import Oracle

    O = Oracle(N, L, A, DB)
    outs = []
    for b in range(x.shape[0]):
        xb, xa = x[b, 0].numpy(), x[b, 1].numpy()
        yb, ya = y[b, 0].numpy(), y[b, 1].numpy()
        ob, oa = O.hmult(LEVEL, xb, xa, yb, ya, evk)
        g = O.gidx(LEVEL - 2)
        outs.append(np.stack([O.canonical(ob, g), O.canonical(oa, g)]).astype(np.int64))
    return torch.from_numpy(np.stack(outs)) if outs else torch.zeros((0, 2, LEVEL - 2, N), dtype=torch.int64)


def _inputs(batch: int):
    from pyoracle import Oracle

    O = Oracle(N, L, A, DB)
    xs, ys = [], []
    for b in range(batch):
        xb, xa, yb, ya, evk = O.synthetic(LEVEL, 900 + b)
        xs.append(np.stack([xb, xa]))
        ys.append(np.stack([yb, ya]))
    return torch.from_numpy(np.stack(xs)), torch.from_numpy(np.stack(ys)), evk


def _worker(rank: int, world: int, port: int, batch: int, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    for p in (os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y, evk = _inputs(batch)
        xy = torch.stack([x, y], dim=1)  # shard x and y together
        out = dp.run_sharded(lambda s: _oracle_hmult_batch(s[:, 0], s[:, 1], evk), xy)
        t = dp.max_over_ranks([float(rank + 1), float(10 * (rank + 1))])
        if rank == 0:
            q.put((out.numpy(), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [3, 4])
def test_sharded_equals_single_rank(batch):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, y, evk = _inputs(batch)
    want = _oracle_hmult_batch(x, y, evk).numpy()
    np.testing.assert_array_equal(got, want)
    assert t == [2.0, 20.0]  # max over ranks


def test_shard_bounds_partition():
    for n in range(0, 17):
        for w in range(1, 9):
            spans = [dp.shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(ValueError):
        dp.shard_bounds(4, 2, 2)


# ---------------------------------------------------------------- on the GPU --
GN, GL, GA, GLEVEL = 1024, 8, 3, 8


def _gpu_worker(rank: int, world: int, port: int, batch: int, q):
    """BASELINE config 3 at N=2 on one GPU: each rank owns a context on cuda:0,
    evaluates HMult+relin and HRot(r=1) of ITS shard through libck32b200
    (the product path, no oracle), results all-gathered over gloo."""
    import sys
    from fractions import Fraction

    here = os.path.dirname(os.path.abspath(__file__))
    for p in (os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_13055_b200 import ckks

        x, y, evk = _gpu_inputs(batch)
        C = ckks.CkksContext(ckks.CkksParams(n=GN, l=GL, alpha=GA, delta_bits=55), device=0)
        relin = ckks.EvaluationKey(torch.from_numpy(evk.astype(np.int32)).cuda(), ckks.RELIN)
        rot = ckks.EvaluationKey(torch.from_numpy(evk.astype(np.int32)).cuda(), ckks.ROTATION, 1)
        s = Fraction(1 << 55)

        def shard_fn(sh):  # [b, 2 (x, y), 2, level, n] -> [b, 2 (hmult, hrot), 2, level, n]
            d = sh.to(torch.int32).cuda()
            X = ckks.Ciphertext(d[:, 0].contiguous(), s, GLEVEL)
            Y = ckks.Ciphertext(d[:, 1].contiguous(), s, GLEVEL)
            m = torch.zeros((sh.shape[0], 2, GLEVEL, GN), dtype=torch.int32, device="cuda")
            m[:, :, : GLEVEL - 2] = ckks.hmult(C, X, Y, relin).data
            r = ckks.hrot(C, X, 1, rot).data
            launches = C.launch_count()
            out = torch.stack([m, r], dim=1).cpu().to(torch.int64)
            assert launches > 0
            return out

        out = dp.run_sharded(shard_fn, torch.stack([x, y], dim=1))
        if rank == 0:
            q.put(out.numpy())
        C.close()
    finally:
        dist.destroy_process_group()


def _gpu_inputs(batch: int):
    from pyoracle import Oracle

    O = Oracle(GN, GL, GA, 55)
    xs, ys = [], []
    for b in range(batch):
        xb, xa, yb, ya, evk = O.synthetic(GLEVEL, 700 + b)
        xs.append(np.stack([xb, xa]))
        ys.append(np.stack([yb, ya]))
    return torch.from_numpy(np.stack(xs)), torch.from_numpy(np.stack(ys)), evk


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [5])
def test_gpu_config3_two_ranks_equal_oracle(batch):
    """2 ranks x cuda:0 (gloo): the gathered HMult / HRot outputs of the
    data-parallel path through libck32b200 equal the oracle's, ciphertext by
    ciphertext (the 2-rank shards are 3 + 2 ciphertexts)."""
    import socket

    from pyoracle import Oracle

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, y, evk = _gpu_inputs(batch)
    O = Oracle(GN, GL, GA, 55)
    for b in range(batch):
        xb, xa, yb, ya = x[b, 0].numpy(), x[b, 1].numpy(), y[b, 0].numpy(), y[b, 1].numpy()
        ob, oa = O.hmult(GLEVEL, xb, xa, yb, ya, evk)
        g = O.gidx(GLEVEL - 2)
        np.testing.assert_array_equal(got[b, 0, :, : GLEVEL - 2], np.stack([O.canonical(ob, g), O.canonical(oa, g)]))
        rb, ra = O.hrot(GLEVEL, xb, xa, 1, evk)
        g = O.gidx(GLEVEL)
        np.testing.assert_array_equal(got[b, 1], np.stack([O.canonical(rb, g), O.canonical(ra, g)]))
