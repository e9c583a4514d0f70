"""Limb-sharded key switching (BASELINE config 4).

CPU tests drive ``limb.LimbShardedEvaluator`` with the oracle-backed shard
(tests/shard_oracle.py, test infrastructure) — in one process (virtual
shards) and over gloo with world size 2 — and compare the reassembled
ciphertexts with the oracle's single-host mechanisms.  GPU tests drive the
native ``ck_shard_*`` path with virtual shards on one B200 and compare with
the single-device mechanisms (themselves pinned to the reference) and with
the reference's full-size hashes at N=2^17 (config 4)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_13055_b200.limb import LimbShardedEvaluator, LocalExchange, ShardLayout, TorchExchange

N, L, A, DB = 256, 6, 2, 55


def _canon(O, a, level):
    return O.canonical(a, O.gidx(level)).astype(np.int64)


def _oracle():
    from pyoracle import Oracle
    return Oracle(N, L, A, DB)


# ---------------------------------------------------------------- layout --
@pytest.mark.parametrize("Lq,alpha", [(6, 2), (24, 8), (8, 3), (54, 14)])
def test_layout_partition(Lq, alpha):
    for world in range(1, 9):
        if world > Lq:
            continue
        lays = [ShardLayout(Lq, alpha, world, r) for r in range(world)]
        assert lays[0].q_lo == 0 and lays[-1].q_hi == Lq
        assert lays[0].p_lo == 0 and lays[-1].p_hi == alpha
        for a, b in zip(lays, lays[1:]):
            assert a.q_hi == b.q_lo and a.p_hi == b.p_lo
        sizes = [x.q_hi - x.q_lo for x in lays]
        assert max(sizes) - min(sizes) <= 1 and max(sizes) == lays[0].q_max
        for level in range(1, Lq + 1):
            assert sum(x.lq(level) for x in lays) == level
            rows = sum((x.q_rows(level) for x in lays), [])
            assert rows == list(range(level))
        full = torch.arange(2 * Lq * 4).reshape(2, Lq, 4)
        assert torch.equal(lays[0].assemble_ct([x.split_ct(full, Lq) for x in lays], Lq), full)


# ------------------------------------------- virtual shards, oracle backend --
def _run_mechanisms(ev, lays, O, level, seed, lazy=False):
    xb, xa, yb, ya, evk = O.synthetic(level, seed)
    x = torch.from_numpy(np.stack([xb, xa]))
    y = torch.from_numpy(np.stack([yb, ya]))
    K = torch.from_numpy(evk)
    xs = [lay.split_ct(x, level) for lay in lays]
    ys = [lay.split_ct(y, level) for lay in lays]
    ks = [lay.split_key(K) for lay in lays]
    got = {}
    got["hmult"] = torch.cat(ev.hmult(level, xs, ys, ks), dim=1).numpy()
    got["hrot1"] = torch.cat(ev.hrot(level, xs, 1, ks), dim=1).numpy()
    got["hrot-3"] = torch.cat(ev.hrot(level, xs, -3, ks), dim=1).numpy()
    got["rescale"] = torch.cat(ev.rescale(level, xs), dim=1).numpy()
    got["ks"] = torch.cat(ev.key_switch(level, [x_[1].contiguous() for x_ in xs], ks), dim=1).numpy()
    want = {}
    lo = level if lazy else level - 2
    ob, oa = O.hmult(level, xb, xa, yb, ya, evk, lazy=lazy)
    want["hmult"] = np.stack([_canon(O, ob, lo), _canon(O, oa, lo)])
    for r in (1, -3):
        ob, oa = O.hrot(level, xb, xa, r, evk)
        want[f"hrot{r}"] = np.stack([_canon(O, ob, level), _canon(O, oa, level)])
    ob, oa = O.rescale(level, xb, xa)
    want["rescale"] = np.stack([_canon(O, ob, level - 2), _canon(O, oa, level - 2)])
    c0, c1 = O.key_switch(level, xa, evk)
    want["ks"] = np.stack([_canon(O, c0, level), _canon(O, c1, level)])
    return got, want


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("lazy", [False, True])
def test_virtual_shards_match_oracle(world, lazy):
    from shard_oracle import OracleShard

    O = _oracle()
    shards = [OracleShard(O, world, r) for r in range(world)]
    ev = LimbShardedEvaluator(shards, LocalExchange(), lazy_rescale=lazy)
    for level, seed in ((L, 31), (4, 32)):
        got, want = _run_mechanisms(ev, [s.layout for s in shards], O, level, seed, lazy)
        for k in want:
            np.testing.assert_array_equal(got[k], want[k], err_msg=f"{k} level {level} world {world}")


# ------------------------------------------------------ gloo, world size 2 --
def _gloo_worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    for p in (os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle"), here):
        if p not in sys.path:
            sys.path.insert(0, p)
    from shard_oracle import OracleShard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = _oracle()
        sh = OracleShard(O, world, rank)
        ev = LimbShardedEvaluator([sh], TorchExchange())
        level = L
        xb, xa, yb, ya, evk = O.synthetic(level, 77)
        x = torch.from_numpy(np.stack([xb, xa]))
        y = torch.from_numpy(np.stack([yb, ya]))
        lay = sh.layout
        k = lay.split_key(torch.from_numpy(evk))
        hm = ev.hmult(level, [lay.split_ct(x, level)], [lay.split_ct(y, level)], [k])[0]
        hr = ev.hrot(level, [lay.split_ct(x, level)], 5, [k])[0]
        q.put((rank, hm.numpy(), hr.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_oracle():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = dict()
    for _ in range(2):
        r, hm, hr = q.get(timeout=300)
        parts[r] = (hm, hr)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = _oracle()
    xb, xa, yb, ya, evk = O.synthetic(L, 77)
    ob, oa = O.hmult(L, xb, xa, yb, ya, evk)
    np.testing.assert_array_equal(np.concatenate([parts[0][0], parts[1][0]], axis=1),
                                  np.stack([_canon(O, ob, L - 2), _canon(O, oa, L - 2)]))
    ob, oa = O.hrot(L, xb, xa, 5, evk)
    np.testing.assert_array_equal(np.concatenate([parts[0][1], parts[1][1]], axis=1),
                                  np.stack([_canon(O, ob, L), _canon(O, oa, L)]))


# ------------------------------------------------------------------- GPU --
def _gpu_ctx(n, l, a, db, lazy=False):
    from paper_2407_13055_b200 import ckks
    return ckks.CkksContext(ckks.CkksParams(n=n, l=l, alpha=a, delta_bits=db, lazy_rescale=lazy))


def _sharded_vs_single(C, O, world, level, seed, lazy=False, rots=(1,), peer=False):
    from fractions import Fraction

    from paper_2407_13055_b200 import ckks
    from paper_2407_13055_b200.limb import LocalPeerExchange, ShardBackend

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(C.device)
    xb, xa, yb, ya, evk = O.synthetic(level, seed)
    x, y, K = dev(np.stack([xb, xa])), dev(np.stack([yb, ya])), dev(evk)
    shards = [ShardBackend(C, world, r) for r in range(world)]
    lays = [s.layout for s in shards]
    xch = LocalPeerExchange(shards) if peer else LocalExchange()
    ev = LimbShardedEvaluator(shards, xch, lazy_rescale=lazy)
    xs = [lay.split_ct(x, level) for lay in lays]
    ys = [lay.split_ct(y, level) for lay in lays]
    ks = [lay.split_key(K) for lay in lays]
    X = ckks.Ciphertext(x, Fraction(1 << O.delta_bits), level)
    Y = ckks.Ciphertext(y, Fraction(1 << O.delta_bits), level)
    got = torch.cat(ev.hmult(level, xs, ys, ks), dim=1)
    want = ckks.hmult(C, X, Y, ckks.EvaluationKey(K))
    assert torch.equal(got, want.data), f"hmult world {world} level {level}"
    for r in rots:
        got = torch.cat(ev.hrot(level, xs, r, ks), dim=1)
        want = ckks.hrot(C, X, r, ckks.EvaluationKey(K, ckks.ROTATION, r))
        assert torch.equal(got, want.data), f"hrot {r} world {world} level {level}"
    if level >= 4:
        got = torch.cat(ev.rescale(level, xs), dim=1)
        assert torch.equal(got, ckks.rescale(C, X).data), f"rescale world {world}"
    got = torch.cat(ev.key_switch(level, [x_[1].contiguous() for x_ in xs], ks), dim=1)
    c0, c1 = ckks.key_switch(C, ckks.Polynomial(x[1].contiguous(), level), ckks.EvaluationKey(K))
    assert torch.equal(got, torch.stack([c0.data, c1.data])), f"key_switch world {world}"
    if peer:
        assert xch.errors() == [0] * world
    for s in shards:
        s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_gpu_virtual_shards_small_vs_oracle_and_single(world, peer):
    from pyoracle import Oracle

    n, l, a, db = 1024, 8, 3, 55
    O = Oracle(n, l, a, db)
    for lazy in (False, True):
        C = _gpu_ctx(n, l, a, db, lazy)
        for level, seed in ((8, 3), (5, 4)):
            _sharded_vs_single(C, O, world, level, seed, lazy, rots=(1, -5), peer=peer)
        C.close()


@pytest.mark.gpu
@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_gpu_virtual_shards_n65536(world, peer):
    from pyoracle import Oracle

    n, l, a, db = 65536, 24, 8, 55
    O = Oracle(n, l, a, db)
    C = _gpu_ctx(n, l, a, db)
    for level in (24, 13):
        _sharded_vs_single(C, O, world, level, 40 + level, peer=peer)
    C.close()


@pytest.mark.gpu
def test_gpu_peer_exchange_rejects_bad_tables_and_times_out():
    """ck_shard_set_peers validates the table; a peer that never signals makes
    the bounded wait report an error instead of hanging the GPU."""
    from paper_2407_13055_b200.limb import ShardBackend

    C = _gpu_ctx(1024, 8, 3, 55)
    shards = [ShardBackend(C, 2, r) for r in range(2)]
    bases = [s.exchange_buffer() for s in shards]
    with pytest.raises(ValueError):
        shards[0].set_peers(bases[:1])  # wrong world size
    with pytest.raises(ValueError):
        shards[0].set_peers([bases[1], bases[1]])  # own entry is not its buffer
    for s in shards:
        s.set_peers(bases)
    shards[0].set_timeout(0.05)
    d = torch.zeros((shards[0].layout.lq(8), 1024), dtype=torch.int32, device=C.device)
    shards[0].modup_begin(8, d, peer=True)  # rank 1 never runs phase 1
    key = shards[0].layout.split_key(torch.zeros((3, 2, 11, 1024), dtype=torch.int32, device=C.device))
    v = shards[0].modup_keymult(8, None, d, key)
    torch.cuda.synchronize()
    assert shards[0].peer_error() == 1
    # the consumer never hands out silently wrong rows: every output word is poison
    assert bool((v == -1).all())
    from paper_2407_13055_b200.limb import LimbShardedEvaluator, LocalPeerExchange

    class _Exch:
        peer = True

        def errors(self):
            return [s.peer_error() for s in shards]

    with pytest.raises(RuntimeError, match="timed out"):
        LimbShardedEvaluator(shards, _Exch()).synchronize()
    # a fresh peer set clears the flag and error words (stale epochs must not
    # satisfy the next wait): rank 1 publishes epoch 1, then the peers are set
    # again; rank 0's wait for epoch 1 must time out again instead of passing
    for s in shards:
        s.set_peers(bases)
    assert shards[0].peer_error() == 0
    shards[1].modup_begin(8, d, peer=True)
    torch.cuda.synchronize()
    for s in shards:
        s.set_peers(bases)
    shards[0].set_timeout(0.05)
    shards[0].modup_begin(8, d, peer=True)
    shards[0].modup_keymult(8, None, d, key)
    torch.cuda.synchronize()
    assert shards[0].peer_error() == 1
    ev = LimbShardedEvaluator(shards, LocalPeerExchange(shards))  # both ranks present: clean
    for s in shards:
        s.set_timeout(10.0)
    x = [torch.zeros((2, s.layout.lq(8), 1024), dtype=torch.int32, device=C.device) for s in shards]
    ev.key_switch(8, [xi[1].contiguous() for xi in x], [key, shards[1].layout.split_key(
        torch.zeros((3, 2, 11, 1024), dtype=torch.int32, device=C.device))])
    ev.synchronize()
    for s in shards:
        s.close()
    C.close()


@pytest.mark.gpu
@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_gpu_config4_n131072_matches_reference_hash(world, peer):
    """BASELINE config 4: single-ciphertext limb-sharded HMult / HRot at
    N=2^17, l=24, alpha=8 — reassembled output equals the reference's hash."""
    from golden_util import FULL, sha
    from pyoracle import Oracle

    from paper_2407_13055_b200.limb import ShardBackend

    cfg = FULL["configs"]["n131072_l24_a8_d55"]
    n, l, a, db = cfg["n"], cfg["l"], cfg["alpha"], cfg["delta_bits"]
    O = Oracle(n, l, a, db)
    C = _gpu_ctx(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(24, FULL["seed"])
    dev = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(C.device)
    x, y, K = dev(np.stack([xb, xa])), dev(np.stack([yb, ya])), dev(evk)
    shards = [ShardBackend(C, world, r) for r in range(world)]
    if peer:
        from paper_2407_13055_b200.limb import LocalPeerExchange
        # the virtual shards run concurrently, one stream each (as on separate GPUs)
        ev = LimbShardedEvaluator(shards, LocalPeerExchange(shards), concurrent=True)
    else:
        ev = LimbShardedEvaluator(shards, LocalExchange())
    lays = [s.layout for s in shards]
    xs = [lay.split_ct(x, 24) for lay in lays]
    ys = [lay.split_ct(y, 24) for lay in lays]
    ks = [lay.split_key(K) for lay in lays]
    hm = torch.cat(ev.hmult(24, xs, ys, ks), dim=1).cpu().numpy()
    assert sha(hm) == cfg["ops"]["hmult@24@0"]
    hr = torch.cat(ev.hrot(24, xs, 1, ks), dim=1).cpu().numpy()
    assert sha(hr) == cfg["ops"]["hrot@24@1"]
    for s in shards:
        s.close()
    C.close()


def _ipc_worker(rank, world, port, q):
    """One shard per process, both on cuda:0: the exchange buffers are mapped
    with CUDA IPC (IpcPeerExchange) exactly as on an NVLink node."""
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    for p in (os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle"), here):
        if p not in sys.path:
            sys.path.insert(0, p)
    from pyoracle import Oracle

    from paper_2407_13055_b200.limb import IpcPeerExchange, ShardBackend

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, l, a, db = 1024, 8, 3, 55
        O = Oracle(n, l, a, db)
        C = _gpu_ctx(n, l, a, db)
        be = ShardBackend(C, world, rank)
        be.set_timeout(60.0)
        xch = IpcPeerExchange(be)
        ev = LimbShardedEvaluator([be], xch)
        dev = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(C.device)
        xb, xa, yb, ya, evk = O.synthetic(l, 91)
        lay = be.layout
        x, y, k = lay.split_ct(dev(np.stack([xb, xa])), l), lay.split_ct(dev(np.stack([yb, ya])), l), \
            lay.split_key(dev(evk))
        out = []
        for _ in range(2):  # repeated exchanges of both kinds: double-buffer reuse
            out.append(ev.hmult(l, [x], [y], [k])[0].cpu().numpy())
            out.append(ev.hrot(l, [x], 3, [k])[0].cpu().numpy())
            out.append(ev.rescale(l, [x])[0].cpu().numpy())
            out.append(ev.rescale(l, [x])[0].cpu().numpy())
        # the same exchanges captured once per rank in a CUDA graph and replayed:
        # the epochs and buffer parities advance on the device
        from paper_2407_13055_b200.pipeline import CapturedStep

        cap = CapturedStep(C.device, lambda: (ev.hmult(l, [x], [y], [k])[0], ev.hrot(l, [x], 3, [k])[0]))
        for _ in range(3):
            m, r = cap.replay()
        torch.cuda.synchronize()
        out.append(m.cpu().numpy())
        out.append(r.cpu().numpy())
        torch.cuda.synchronize()
        q.put((rank, out, xch.errors()))
        dist.barrier()
        xch.close()
        be.close()
        C.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_ipc_peer_exchange_two_processes():
    """Config 4's peer-memory exchange across processes (CUDA IPC, flags with
    system-scope release / acquire): both ranks share cuda:0 here; the same
    code maps NVLink peers on a multi-GPU node.  Bit-exact vs the oracle,
    eagerly and replayed from a CUDA graph captured on each rank."""
    from pyoracle import Oracle

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = {}
    for _ in range(2):
        r, out, err = q.get(timeout=600)
        assert err == [0]
        parts[r] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, l, a, db = 1024, 8, 3, 55
    O = Oracle(n, l, a, db)
    xb, xa, yb, ya, evk = O.synthetic(l, 91)
    ob, oa = O.hmult(l, xb, xa, yb, ya, evk)
    hm = np.stack([_canon(O, ob, l - 2), _canon(O, oa, l - 2)])
    ob, oa = O.hrot(l, xb, xa, 3, evk)
    hr = np.stack([_canon(O, ob, l), _canon(O, oa, l)])
    ob, oa = O.rescale(l, xb, xa)
    rs = np.stack([_canon(O, ob, l - 2), _canon(O, oa, l - 2)])
    for i, want in enumerate([hm, hr, rs, rs] * 2 + [hm, hr]):
        got = np.concatenate([parts[0][i], parts[1][i]], axis=1).astype(np.int64)
        np.testing.assert_array_equal(got, want)
